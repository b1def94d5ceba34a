"""Debug helper: one tensor-parallel verify (torchrun, one GPU per rank) of a synthetic batch.
  torchrun --nproc-per-node 2 tools/dbg_tp.py ; env SHAPE="layers,d,heads,kv,hd,ffn,vocab",
  B, CTX_LO, CTX_HI, NODES, FUSED=0/1.  GPU only."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_17052_b200 import api  # noqa: E402
from synth.configs import ModelShape  # noqa: E402
from synth.trees import pooled_tree  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
    L_, d, H, KV, hd, F, V = (int(x) for x in os.environ.get("SHAPE", "2,1024,16,2,128,2048,4096").split(","))
    shape = ModelShape("dbg", L_, d, H, KV, hd, F, V, 1e-5, 500000.0)
    obj = [api.tp_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, 0)
    rng = np.random.default_rng(909)
    B = int(os.environ.get("B", "8"))
    ctx = [int(x) for x in rng.integers(int(os.environ.get("CTX_LO", "3072")), int(os.environ.get("CTX_HI", "5120")) + 1, B)]
    sizes = [int(os.environ.get("NODES", "64"))] * B
    maxc = max(ctx) + 128
    model = api.Model(shape, 3, device=rank, max_position=maxc + 64, tp_rank=rank, tp_size=world, nccl_id=obj[0])
    trees = [pooled_tree(rng, n, 8, 4, shape.vocab) for n in sizes]
    R = sum(t.n + 1 for t in trees)
    if os.environ.get("FUSED", "0") == "1":
        model.tp_fused_enable(R)
    pool = api.KVPool(model, sum((c + 127) // 64 for c in ctx) + 8, B)
    hs = []
    for r in range(B):
        h = pool.alloc(ctx[r] + 80)
        pool.fill_random(h, ctx[r] - 1, 4321, r)
        hs.append(h)
    ws = model.workspace(B, R, maxc)
    batch = api.Batch.from_host(hs, ctx, [1] * B, [2000 + r for r in range(B)], [0] * B, trees,
                                device=f"cuda:{rank}", max_context_len=maxc)
    out = api.verify(model, pool, batch, ws, auto_commit=False)
    torch.cuda.synchronize()
    rt = out.row_target.cpu().numpy()
    rs = out.row_score.cpu().numpy().astype(np.float64)
    print(f"rank {rank}: ok, accepted {out.accepted_len.cpu().numpy().tolist()[:8]} target_sum {int(rt.sum())} "
          f"score_mean {rs.mean():.6f}", flush=True)
    model.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
