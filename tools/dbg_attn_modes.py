"""Debug helper: run one verify of the long-ragged-context scenario and print which rows of the
final logits are non-finite (run with and without SPECEDGE_ATTN_BALANCED=1).  GPU only."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_17052_b200 import api  # noqa: E402
from synth.configs import SMALL128  # noqa: E402
from synth.trees import pooled_tree  # noqa: E402


def main():
    shape = SMALL128
    rng = np.random.default_rng(909)
    ctx = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "4500,200,7000,4100,64".split(","))]
    sizes = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "16,32,8,63,1".split(","))]
    B = len(ctx)
    model = api.Model(shape, 3, max_position=8192)
    pool = api.KVPool(model, sum((c + 127) // 64 for c in ctx) + 8, B)
    hs = []
    for r in range(B):
        h = pool.alloc(ctx[r] + 64)
        pool.fill_random(h, ctx[r] - 1, 4321, r)
        hs.append(h)
    trees = [pooled_tree(rng, n, 5, 3, shape.vocab) for n in sizes]
    ws = model.workspace(B, sum(t.n + 1 for t in trees), 7100)
    batch = api.Batch.from_host(hs, ctx, [1] * B, [2000 + r for r in range(B)], [0] * B, trees, max_context_len=7100)
    api.verify(model, pool, batch, ws, auto_commit=False)
    lg = api.debug_last_logits(model, ws, batch).cpu().numpy()
    bad = np.where(~np.isfinite(lg).all(axis=1))[0]
    off = np.cumsum([0] + [t.n + 1 for t in trees])
    print("rows", lg.shape[0], "bad rows", bad.tolist(), "request offsets", off.tolist())
    np.save(os.environ.get("OUT", "gpurun_out/lg.npy"), lg)


if __name__ == "__main__":
    main()
