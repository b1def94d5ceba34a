"""Debug helper: one verify of a synthetic batch on one GPU, printing which rows of the final
logits are non-finite (run with and without SPECEDGE_ATTN_BALANCED=1).  GPU only.
  python tools/dbg_attn_modes.py [ctx,ctx,...] [nodes,nodes,...]
  SHAPE="layers,d,heads,kv,hd,ffn,vocab" (default small128), B/CTX_LO/CTX_HI/NODES for a random batch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_17052_b200 import api  # noqa: E402
from synth.configs import SMALL128, ModelShape  # noqa: E402
from synth.trees import pooled_tree  # noqa: E402


def main():
    shape = SMALL128
    if os.environ.get("SHAPE"):
        L_, d, H, KV, hd, F, V = (int(x) for x in os.environ["SHAPE"].split(","))
        shape = ModelShape("dbg", L_, d, H, KV, hd, F, V, 1e-5, 500000.0)
    rng = np.random.default_rng(909)
    if os.environ.get("B"):
        B = int(os.environ["B"])
        ctx = [int(x) for x in rng.integers(int(os.environ["CTX_LO"]), int(os.environ["CTX_HI"]) + 1, B)]
        sizes = [int(os.environ.get("NODES", "64"))] * B
    else:
        ctx = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4500,200,7000,4100,64").split(",")]
        sizes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16,32,8,63,1").split(",")]
    B = len(ctx)
    maxc = max(ctx) + 128
    model = api.Model(shape, 3, max_position=maxc + 64)
    pool = api.KVPool(model, sum((c + 127) // 64 for c in ctx) + 8, B)
    hs = []
    for r in range(B):
        h = pool.alloc(ctx[r] + 64)
        pool.fill_random(h, ctx[r] - 1, 4321, r)
        hs.append(h)
    trees = [pooled_tree(rng, n, 7, 4, shape.vocab) for n in sizes]
    ws = model.workspace(B, sum(t.n + 1 for t in trees), maxc)
    batch = api.Batch.from_host(hs, ctx, [1] * B, [2000 + r for r in range(B)], [0] * B, trees, max_context_len=maxc)
    api.verify(model, pool, batch, ws, auto_commit=False)
    torch.cuda.synchronize()
    lg = api.debug_last_logits(model, ws, batch).cpu().numpy()
    bad = np.where(~np.isfinite(lg).all(axis=1))[0]
    off = np.cumsum([0] + [t.n + 1 for t in trees])
    print("rows", lg.shape[0], "bad rows", bad.tolist()[:20], "request offsets", off.tolist()[:8])
    np.save(os.environ.get("OUT", "gpurun_out/lg.npy"), lg)


if __name__ == "__main__":
    main()
