"""Model shapes and workload presets (inputs only, no arithmetic).

Shapes follow SURVEY.md Appendix B (public HF config values for the model families the
paper evaluates).  Workload presets follow BASELINE.json `configs`
and SURVEY.md §8(d).
"""
from __future__ import annotations

from dataclasses import dataclass, replace, asdict


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d: int
    n_heads: int
    n_kv: int
    head_dim: int
    ffn: int
    vocab: int
    eps: float
    rope_theta: float

    @property
    def group(self) -> int:
        return self.n_heads // self.n_kv

    def as_dict(self):
        return asdict(self)


# cfg1: tiny decoder (BASELINE.json configs[0]; SURVEY.md amb. A24 fixes kv-heads, hd, F, theta, eps)
TINY = ModelShape("tiny", 2, 64, 4, 2, 16, 256, 256, 1e-6, 10000.0)
# tiny with V=16 for the chi-square law test
TINY_V16 = replace(TINY, name="tiny-v16", vocab=16)
# tiny MHA variant (kv = heads) used to exercise G = 1
TINY_MHA = replace(TINY, name="tiny-mha", n_kv=4)
# cfg2: Llama-3-8B-shaped
LLAMA3_8B = ModelShape("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256, 1e-5, 500000.0)
# 2-layer slice of the cfg2 shape at full width / full vocab, for full-size sampled parity
LLAMA3_8B_2L = replace(LLAMA3_8B, name="llama3-8b-2l", n_layers=2)
# cfg3 / cfg5: Qwen3-14B-shaped (QK-norm off, SURVEY.md amb. A16)
QWEN3_14B = ModelShape("qwen3-14b", 40, 5120, 40, 8, 128, 17408, 151936, 1e-6, 1000000.0)
# 2-layer slice of the cfg3 / cfg5 shape at full width / full vocab (parity at bench widths)
QWEN3_14B_2L = replace(QWEN3_14B, name="qwen3-14b-2l", n_layers=2)
# cfg4: Llama-3-70B-shaped
LLAMA3_70B = ModelShape("llama3-70b", 80, 8192, 64, 8, 128, 28672, 128256, 1e-5, 500000.0)
# the paper's edge draft models are Qwen3-0.6B / 1.7B; NEXT-F3 timing uses this shape
QWEN3_0_6B = ModelShape("qwen3-0.6b", 28, 1024, 16, 8, 128, 3072, 151936, 1e-6, 1000000.0)
# a small hd=128 model used by GPU unit tests (fast, exercises the hd=128 kernels)
SMALL128 = ModelShape("small128", 2, 512, 8, 2, 128, 1024, 2048, 1e-5, 500000.0)

SHAPES = {s.name: s for s in (TINY, TINY_V16, TINY_MHA, LLAMA3_8B, LLAMA3_8B_2L,
                              QWEN3_14B, QWEN3_14B_2L, LLAMA3_70B, SMALL128, QWEN3_0_6B)}


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config restated as per-GPU shapes."""
    name: str
    shape: ModelShape
    weight_seed: int
    n_requests: int
    n_nodes: int          # draft nodes per tree, root excluded (SURVEY.md amb. A1)
    depth: int            # draft passes D
    branching: int        # b
    ctx_lo: int           # committed context length C_r ~ U[ctx_lo, ctx_hi]
    ctx_hi: int
    ctx_seed: int
    accept_mu: float      # planted tokens/verify profile (accepted + bonus), Table 1 means
    accept_sigma: float
    mode: str             # "greedy" | "sample"
    temperature: float
    real_prefill: bool    # parity configs prefill for real; perf configs random-fill KV
    tp: bool = False      # one tensor-parallel model over all ranks (cfg4) instead of per-GPU replicas
    microbatches: int = 1  # resident request sets per GPU verified alternately (cfg3: A/B)


CFG1 = Workload("cfg1", TINY, 1, 1, 8, 4, 3, 32, 32, 101, 3.98, 1.55, "greedy", 0.0, True)
CFG2 = Workload("cfg2", LLAMA3_8B, 2, 16, 32, 7, 4, 768, 1280, 102, 3.98, 1.55, "greedy", 0.0, False)
CFG3 = Workload("cfg3", QWEN3_14B, 3, 32, 32, 7, 4, 1536, 2560, 103, 4.44, 2.1, "greedy", 0.0, False,
                microbatches=2)
CFG5 = Workload("cfg5", QWEN3_14B, 5, 16, 16, 5, 4, 12288, 20480, 105, 3.98, 1.55, "sample", 1.0, False)
# cfg4: Llama-3-70B-shaped, tensor parallel over the box's GPUs (TP = 8 in BASELINE.json; any
# divisor of 8 heads runs), 32 requests for the whole box
CFG4 = Workload("cfg4", LLAMA3_70B, 4, 32, 64, 8, 4, 3072, 5120, 104, 4.67, 2.6, "greedy", 0.0, False, tp=True)

WORKLOADS = {w.name: w for w in (CFG1, CFG2, CFG3, CFG4, CFG5)}
