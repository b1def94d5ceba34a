"""Tensor-parallel verify (SURVEY §8(a) a12, §8(e) TP regime; P14 "TP = k == TP = 1"): TP
processes, one GPU each, run the same verify through specedge_model_create_tp shards with the
collectives C1/C2 (reduce-scatter after O and down: NCCL, or the NEXT-F4 GEMM epilogues pushing
into the owners' NVLink-mapped receive slots) and C3 (all-gather of per-row winners).  Checked
against the oracle exactly as the TP = 1 parity tests are (tests/gpu_helpers.py contract):
concatenated vocab-shard logits, per-slot targets, the walk on the library's own targets,
acceptance outputs, and on every rank the committed KV of its kv-head shard equal bit for bit to
its tree-scratch rows of the accepted slots (plus close to the oracle cache slice).  TP = 2 / 4 / 8
need that many GPUs (gpurun --gpus N); the sharding itself is checked on one GPU by
tests/test_gpu_tp_shards.py."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import verify as OV  # noqa: E402
from oracle.model import Weights  # noqa: E402
from synth.configs import ModelShape  # noqa: E402
from synth.plant import plant, draw_accept_lengths  # noqa: E402
from synth.trees import pooled_tree  # noqa: E402
from tests.gpu_helpers import (check_batch, check_commit, check_logits, f16_bits_to_f64,  # noqa: E402
                               oracle_noise_floor, split_outputs)

SEED = 7
# SURVEY App. B "tiny-tp": 8 q / 8 kv heads of 128 so that TP = 2, 4 and 8 all shard it
TINY_TP = ModelShape("tiny-tp", 2, 1024, 8, 8, 128, 2048, 1024, 1e-6, 10000.0)


def _needs_gpus(n):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")


def _setup(seed=SEED):
    """Host-side inputs shared by every rank and the oracle (a pure function of the seed)."""
    shape = TINY_TP
    rng = np.random.default_rng(909)
    B = 4
    prompts = [[int(t) for t in rng.integers(0, shape.vocab, n)] for n in (40, 75, 17, 64)]
    W = Weights(shape, seed)
    sessions = [OV.make_session(W, p, 300 + i) for i, p in enumerate(prompts)]
    trees = [pooled_tree(rng, n, 4, 3, shape.vocab) for n in (8, 32, 16, 4)]
    a = draw_accept_lengths(rng, trees, 3.98, 1.55)

    def targets(trs):
        return [OV.verify_one(W, OV.Request(sessions[i], t.parent, t.token), keep_logits=False).row_target
                for i, t in enumerate(trs)]
    trees = plant(trees, targets, a, shape.vocab, rng)
    return shape, W, prompts, sessions, trees


def _worker(rank, tp, nccl_id, mode, temperature, q, fused=False):
    try:
        torch.cuda.set_device(rank)
        from paper_2505_17052_b200 import api
        shape, W, prompts, sessions, trees = _setup()
        model = api.Model(shape, SEED, device=rank, max_position=4096, tp_rank=rank, tp_size=tp, nccl_id=nccl_id)
        if fused:   # NEXT-F4: "push" (epilogue bulk copies into the owners' receive slots) or "nvls"
            model.tp_fused_enable(4 * 65)
            assert model.tp_fused_mode() == fused, model.tp_fused_mode()
        cap = max(len(p) for p in prompts) + 256
        pool = api.KVPool(model, ((cap + 63) // 64) * len(prompts) + 4, len(prompts) + 4)
        B = len(prompts)
        ws = model.workspace(B, B * 65, cap)
        handles = []
        for p in prompts:
            h = pool.alloc(cap)
            pool.prefill(h, p, ws)
            handles.append(h)
        L0 = [int(x) for x in pool.get_len(handles)]
        batch = api.Batch.from_host(handles, [s.context_len for s in sessions], [s.last_token for s in sessions],
                                    [s.session_id for s in sessions], [s.round for s in sessions], trees,
                                    max_context_len=max(s.context_len for s in sessions) + 8)
        mode_c = api.L.GREEDY if mode == "greedy" else api.L.SAMPLE_TREE
        out = api.verify(model, pool, batch, ws, mode=mode_c, temperature=temperature, seed=SEED, auto_commit=True)
        logits = api.debug_last_logits(model, ws, batch).cpu().numpy()
        torch.cuda.synchronize()
        g = split_outputs(out, batch)
        # this rank's kv-head shard: committed rows == its tree-scratch rows of the accepted slots
        check_commit(api, model, pool, ws, batch, g, handles, L0)
        res = dict(g=g, status=out.status.cpu().numpy(), accepted_len=out.accepted_len.cpu().numpy(),
                   accepted_token=out.accepted_token.cpu().numpy(), accepted_node=out.accepted_node.cpu().numpy(),
                   bonus=out.bonus.cpu().numpy(), row_target=out.row_target.cpu().numpy(),
                   row_score=out.row_score.cpu().numpy(), logits=logits, vocab0=model.vocab0,
                   lens=pool.get_len(handles))
        res["kv"] = [[pool.read_kv(h, l, sel, 0, int(res["lens"][i])) for l in range(shape.n_layers)
                      for sel in (0, 1)] for i, h in enumerate(handles)]
        pool.close()
        model.close()
        q.put((rank, res))
    except Exception as e:  # surfaced by the parent
        import traceback
        q.put((rank, RuntimeError(f"rank {rank}: {e}\n{traceback.format_exc()}")))


def _run_tp(tp, mode, temperature, fused=False):
    import torch.multiprocessing as mp
    from paper_2505_17052_b200 import api
    nccl_id = api.tp_unique_id()
    if fused == "nvls":   # read by the spawned workers' library at tp_fused_enable
        os.environ["SPECEDGE_TP_F4"] = "nvls"
    else:
        os.environ.pop("SPECEDGE_TP_F4", None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, tp, nccl_id, mode, temperature, q, fused)) for r in range(tp)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(tp):
        r, v = q.get(timeout=600)
        if isinstance(v, Exception):
            raise v
        res[r] = v
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("tp", [2, 4, 8])
@pytest.mark.parametrize("mode,temperature,fused", [("greedy", 0.0, False), ("sample", 1.0, False),
                                                   ("greedy", 0.0, "push"), ("sample", 1.0, "push"),
                                                   ("greedy", 0.0, "nvls"), ("sample", 1.0, "nvls")])
def test_tp_verify_matches_oracle(tp, mode, temperature, fused):
    """fused: NEXT-F4 GEMM -> reduce-scatter over NVLink peer memory ("push") or through an NVLS
    multicast object with in-switch reduction ("nvls") instead of NCCL for C1/C2."""
    _needs_gpus(tp)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    res = _run_tp(tp, mode, temperature, fused)
    shape, W, prompts, sessions, trees = _setup()
    B = len(prompts)
    refs = OV.verify_batch(W, [OV.Request(sessions[r], trees[r].parent, trees[r].token) for r in range(B)],
                           mode=mode, temperature=temperature, seed=SEED, auto_commit=True)
    # replicated outputs: identical on every rank
    for rank in range(1, tp):
        for k in ("status", "accepted_len", "accepted_token", "accepted_node", "bonus", "row_target", "row_score"):
            assert np.array_equal(res[0][k], res[rank][k]), (rank, k)
    # vocab shards concatenate to the full logits
    assert res[0]["vocab0"] == 0
    for rank in range(1, tp):
        assert res[rank]["vocab0"] == res[rank - 1]["vocab0"] + res[rank - 1]["logits"].shape[1]
    logits = np.concatenate([res[rank]["logits"] for rank in range(tp)], axis=1)
    ref_logits = np.concatenate([o.logits for o in refs])
    def run():
        ses2 = _setup()[3]
        return np.concatenate([o.logits for o in OV.verify_batch(
            W, [OV.Request(ses2[r], trees[r].parent, trees[r].token) for r in range(B)], mode=mode,
            temperature=temperature, seed=SEED, auto_commit=False)])
    bound = check_logits(logits, ref_logits, noise_fn=lambda: oracle_noise_floor(run)[1])
    g = res[0]["g"]
    assert all(int(x) == 0 for x in g["status"])
    # the oracle committed (round advanced): score with the round the verify used
    scores = [OV.target_scores(o.logits, mode, temperature, SEED, sessions[r].round - 1, sessions[r].session_id)
              for r, o in enumerate(refs)]
    invT = OV.inv_temperature(temperature) if temperature else 1.0
    kinds = check_batch(trees, refs, scores, g, bound * invT + 1e-5)
    # committed KV values: each rank holds kv heads [rank*KV/TP, (rank+1)*KV/TP) of the oracle cache
    kvl = shape.n_kv // tp
    for r in range(B):
        if kinds[r] != "exact":
            continue
        ses = sessions[r]
        assert int(res[0]["lens"][r]) == len(ses.cache)
        for rank in range(tp):
            for l in range(shape.n_layers):
                for sel, ref in ((0, ses.cache.k[l]), (1, ses.cache.v[l])):
                    got = f16_bits_to_f64(res[rank]["kv"][r][2 * l + sel])
                    want = ref[:, rank * kvl:(rank + 1) * kvl]
                    num = np.linalg.norm((got - want).reshape(len(want), -1), axis=1)
                    den = np.linalg.norm(want.reshape(len(want), -1), axis=1)
                    assert (num / np.maximum(den, 1e-30)).max() <= 2e-2, (r, rank, l, sel)
