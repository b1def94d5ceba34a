"""Step time of the three verify modes on cfg2 shapes (Llama-3-8B-shaped, 16 requests, 528 rows):
GREEDY and SAMPLE_TREE on 32-node trees, SAMPLE_PQ_DENSE (NEXT-F2) on 32-node sampled chains with
dense q rows (16 x 32 x 128256 fp32 = 263 MB of draft distributions).  Prints one JSON line per mode
(device time per verify step, CUDA events over graph-replayed steps).  GPU only.
Usage: python tools/pq_timing.py [--steps 20]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import setup_gpu  # noqa: E402
from synth.configs import CFG2  # noqa: E402
from synth.trees import Tree  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    st = setup_gpu(CFG2, 0, 0)
    api, model, pool, ws, batch = st["api"], st["model"], st["pool"], st["ws"], st["batch"]
    handles, L0 = st["handles"], [c - 1 for c in st["ctx"]]
    V = CFG2.shape.vocab
    rng = np.random.default_rng(3)
    chains = [Tree(np.arange(-1, 31, dtype=np.int32), rng.integers(0, V, 32).astype(np.int32),
                   np.zeros(32, np.float32)) for _ in range(CFG2.n_requests)]
    cb = api.Batch.from_host(handles, st["ctx"], batch.root_token.cpu().numpy(), batch.session_id.cpu().numpy(),
                             [0] * CFG2.n_requests, chains, max_context_len=batch.max_context_len)
    q = torch.rand((cb.total_nodes, V), device="cuda", dtype=torch.float32)
    cb.draft_q = q / q.sum(dim=1, keepdim=True)
    cases = [("greedy", batch, api.L.GREEDY, 0.0), ("sample_tree", batch, api.L.SAMPLE_TREE, 1.0),
             ("pq_dense", cb, api.L.SAMPLE_PQ_DENSE, 1.0)]
    for name, b, mode, T in cases:
        out = api.Outputs.alloc(b, "cuda")

        def step():
            api.verify(model, pool, b, ws, mode=mode, temperature=T, seed=7, auto_commit=True, out=out)
            pool.set_len(handles, L0)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        # per-kernel split of one extra (event-instrumented) step
        import ctypes as C
        lib = model.lib
        nk = len(api.L.KERNEL_KINDS)
        lib.specedge_kernel_times(None, None, 1)
        lib.specedge_set_kernel_timing(-1)
        step()
        torch.cuda.synchronize()
        lib.specedge_set_kernel_timing(0)
        kms, kc = (C.c_float * nk)(), (C.c_int32 * nk)()
        lib.specedge_kernel_times(kms, kc, 1)
        split = {api.L.KERNEL_KINDS[i]: round(float(kms[i]), 3) for i in range(nk) if kc[i] and kms[i] > 0.05}
        acc = out.accepted_len.cpu().numpy()
        st_codes = out.status.cpu().numpy()
        print(json.dumps({"mode": name, "ms_per_step": round(ms, 4), "rows": b.rows,
                          "tokens_per_step": int((acc + 1).sum()), "status_ok": int((st_codes == 0).sum()),
                          "kernels_ms": split}),
              flush=True)


if __name__ == "__main__":
    main()
