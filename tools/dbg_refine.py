"""Debug: candidate statistics and timing of the hi-only LM head refinement on a bench config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_17052_b200 import api
from synth.configs import WORKLOADS
from synth.trees import pooled_tree
wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
if len(sys.argv) > 2:   # override the mode: greedy / sample
    import dataclasses
    wl = dataclasses.replace(wl, mode=sys.argv[2], temperature=1.0 if sys.argv[2] == "sample" else 0.0)
rng = np.random.default_rng(1)
B = wl.n_requests
ctx = [int(c) for c in rng.integers(wl.ctx_lo, wl.ctx_hi + 1, B)]
cap = max(ctx) + wl.n_nodes + 64
model = api.Model(wl.shape, wl.weight_seed, max_position=cap + 64)
pool = api.KVPool(model, sum((c + wl.n_nodes + 127) // 64 for c in ctx) + 4, B)
hs = []
for r, c in enumerate(ctx):
    h = pool.alloc(c + wl.n_nodes + 64); pool.fill_random(h, c - 1, 5, r); hs.append(h)
trees = [pooled_tree(rng, wl.n_nodes, wl.depth, wl.branching, wl.shape.vocab) for _ in range(B)]
ws = model.workspace(B, sum(t.n + 1 for t in trees), cap)
batch = api.Batch.from_host(hs, ctx, [1] * B, list(range(B)), [0] * B, trees, max_context_len=cap)
for _ in range(3):
    out = api.verify(model, pool, batch, ws, mode=1 if wl.mode == "sample" else 0, temperature=wl.temperature,
                     seed=3, auto_commit=False)
torch.cuda.synchronize()
lib = model.lib
import ctypes as C
nk = len(api.L.KERNEL_KINDS)
lib.specedge_kernel_times(None, None, 1)
lib.specedge_set_kernel_timing(-1)
for _ in range(5):
    api.verify(model, pool, batch, ws, mode=1 if wl.mode == "sample" else 0, temperature=wl.temperature, seed=3,
               auto_commit=False)
torch.cuda.synchronize()
lib.specedge_set_kernel_timing(0)
ms = (C.c_float * nk)(); cnt = (C.c_int32 * nk)()
lib.specedge_kernel_times(ms, cnt, 1)
for i, k in enumerate(api.L.KERNEL_KINDS):
    if cnt[i]:
        print(f"{k:14s} {ms[i] / 5:8.4f} ms/step  launches {cnt[i] // 5}")
