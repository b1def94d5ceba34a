"""Mainloop throughput probe of the tcgen05 GEMM (debug entry point, fp32-store epilogue).
One tile per CTA: M = 148*128 weight rows, R = BN activation rows, K large -> time per k-block
tells whether the k-loop is MMA-bound (2*BN cycles per 64-deep k-block at M=128) or bound by
operand delivery (bytes per k-block per SM = 16 KB + BN*128 B)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_17052_b200 import api

torch.manual_seed(0)
res = []
for (M, R, K) in [(148 * 128, 64, 8192), (148 * 128, 128, 8192), (148 * 128, 176, 8192), (148 * 128, 256, 8192),
                  (148 * 128 * 2, 256, 8192), (4096, 528, 4096), (6144, 528, 4096), (28672, 528, 4096),
                  (4096, 528, 14336), (128256, 1056, 4096)]:
    W = (torch.randn(M, K, device="cuda") / 64).to(torch.bfloat16)
    X = torch.randn(R, K, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        api.debug_gemm(W, X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        api.debug_gemm(W, X)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = 2.0 * M * R * K
    kb = K // 64
    tiles = ((M + 127) // 128) * ((R + 255) // 256)
    r = dict(M=M, R=R, K=K, us=round(ms * 1e3, 2), tflops=round(fl / ms / 1e9, 1),
             us_per_kblock_per_tile=round(ms * 1e3 / kb / max(1, tiles / 148), 4))
    res.append(r)
    print(json.dumps(r), flush=True)
    del W, X
