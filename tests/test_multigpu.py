"""N > 1 path on CPU (per-GPU replicas, no collective on the data path).
world_size-2 gloo process groups stand in for the NCCL ranks: the only cross-rank operations of the
benchmark are the barrier, the max-over-ranks timing reduction and the sum of the replicas' verified tokens; the data path itself must be
independent of placement (a request verified on any rank gives the same outcome)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import verify as OV
    from oracle.model import Weights
    from synth.configs import CFG2, TINY
    from synth.trees import pooled_tree
    # 1) timing aggregation: max over ranks, whole-box throughput
    local_ms = 100.0 + 50.0 * rank
    mx = bench.reduce_max(local_ms, dist)
    dist.barrier()
    # 2) placement independence: every rank verifies the same request (same session id, seed)
    rng = np.random.default_rng(7)
    W = Weights(TINY, 1)
    prompt = [int(t) for t in rng.integers(0, TINY.vocab, 20)]
    ses = OV.make_session(W, prompt, 1234)
    tree = pooled_tree(rng, 8, 4, 3, TINY.vocab)
    o = OV.verify_one(W, OV.Request(ses, tree.parent, tree.token), "sample", 0.7, 99)
    # 3) per-rank workloads differ (replicas verify different requests)
    ctx = bench.contexts(CFG2, rank)
    # tokens verified per step differ per replica (70 on rank 0, 74 on rank 1): summed over ranks
    box_tokens = bench.reduce_sum(70 + 4 * rank, dist)
    q.put((rank, mx, bench.box_throughput(box_tokens, 10, mx), o.accepted_token, o.bonus, ctx))
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, mx0, v0, acc0, b0, c0), (r1, mx1, v1, acc1, b1, c1) = res
    assert mx0 == mx1 == 150.0                       # slowest rank's clock
    assert v0 == v1 == pytest.approx((70 + 74) * 10 / 0.150)
    assert (acc0, b0) == (acc1, b1)                  # same request -> same outcome on any rank
    assert c0 != c1                                  # replicas own different requests


def test_bench_acceptance_profile_is_the_table1_mean_on_every_rank():
    """The bench plants acceptance lengths whose request-set total is round((mu - 1) B) on every rank
    (Table 1 profile mean), within each tree's depth; the spread of the normal draw stays."""
    from synth.configs import WORKLOADS
    from synth.plant import draw_accept_lengths_at_mean
    import bench
    for name in ("cfg2", "cfg3", "cfg5", "cfg4"):
        wl = WORKLOADS[name]
        for rank in range(4):
            trees = bench.build_trees(wl, rank, wl.shape.vocab)
            a = draw_accept_lengths_at_mean(np.random.default_rng([wl.ctx_seed + 11, rank]), trees, wl.accept_mu,
                                            wl.accept_sigma)
            assert sum(a) == int(round((wl.accept_mu - 1.0) * wl.n_requests)), (name, rank, a)
            assert all(0 <= x <= int(t.depth().max()) for x, t in zip(a, trees))
            assert len(set(a)) > 1
