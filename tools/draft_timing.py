"""NEXT-F3 timing: build draft trees (budget 32, depth 7, branching 4 — the paper's tree shape,
P:599) with a Qwen3-0.6B-shaped random-init draft model (the paper's edge draft) on a B200,
context ~1k tokens.  Prints one JSON line: ms per tree, passes, nodes.  GPU only."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_17052_b200 import api  # noqa: E402
from synth.configs import QWEN3_0_6B  # noqa: E402


def main():
    shape = QWEN3_0_6B
    model = api.Model(shape, 21, max_position=4096)
    pool = api.KVPool(model, 40, 4)
    h = pool.alloc(1100)
    pool.fill_random(h, 1023, 21, 0)
    ws = model.workspace(1, 33, 1100)
    root = 17
    for _ in range(2):
        api.draft_tree(model, pool, h, 1024, root, 5, 32, 7, 4, ws)
    torch.cuda.synchronize()
    n = 10
    t0 = time.perf_counter()
    for _ in range(n):
        par, tok, lp = api.draft_tree(model, pool, h, 1024, root, 5, 32, 7, 4, ws)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / n
    depth = np.zeros(len(par), int)
    for i, p in enumerate(par):
        depth[i] = 1 if p < 0 else depth[p] + 1
    print(json.dumps({"draft_model": shape.name, "budget": 32, "depth": 7, "branching": 4, "ms_per_tree": round(ms, 3),
                      "nodes": int(len(par)), "max_depth": int(depth.max()), "context": 1024}))


if __name__ == "__main__":
    main()
