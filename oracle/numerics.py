"""Elementwise numerics of the target decoder, float64.

Precision reading (DESIGN.md R-precision, revising SURVEY amb. A12; the paper states no precision
anywhere, P:16/P:744 only quote marketing TFLOPS): bf16-valued are weights, embeddings and the
GEMM input operands (normed h, attention output O, MLP hidden M); fp16-valued are the attention
operands q, k (post-RoPE) and v, i.e. also the KV cache; the residual stream and the final-norm
output are not rounded.  `bf16` below rounds an exact (float64) value to the nearest bf16 value,
ties to even.  All other arithmetic is float64.
"""
from __future__ import annotations

import numpy as np


def bf16(x):
    """Round to nearest bfloat16 (8 significant bits, 8-bit exponent), ties to even.

    x = m * 2**e with m in [0.5, 1); bf16 spacing at x is 2**(e-8), or the subnormal spacing
    2**-133 below 2**-126.  Division/multiplication by powers of two is exact in float64 and
    np.rint rounds half to even.  Pinned against torch's fp32->bf16 converter.
    """
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    e = np.maximum(e - 8, -133)
    spacing = np.ldexp(1.0, e)
    y = np.rint(x / spacing) * spacing
    y = np.where(np.abs(y) >= 2.0 ** 128, np.copysign(np.inf, x), y)   # overflow past bf16 max
    return np.where(np.isfinite(x), y, x)


def f16(x):
    """Round to nearest IEEE binary16 (11 significant bits, subnormals below 2^-14), ties to even,
    overflow to inf.  Same construction as `bf16`; pinned against numpy's float16 conversion."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    e = np.maximum(e - 11, -24)
    spacing = np.ldexp(1.0, e)
    y = np.rint(x / spacing) * spacing
    y = np.where(np.abs(y) >= 65520.0, np.copysign(np.inf, x), y)
    return np.where(np.isfinite(x), y, x)


def f32(x):
    """Round to float32 (IEEE RNE), returned as float64."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


# Noise-floor estimation (test infrastructure, off unless a test sets it): (rng, eps).  Every
# activation storage point (model.py: h, q, k, v, O, M; attention_weights: P) first scales its
# input by (1 + eps * U(-1, 1)) — an implementation whose fp32 arithmetic (summation order,
# approximate exp2 / rsqrt, tensor-core accumulation) lands within eps of the exact pre-rounding
# values.  Weights, embeddings and synthetic caches are never perturbed.
PERTURB = None


def perturb(x):
    if PERTURB is None:
        return x
    rng, eps = PERTURB
    x = np.asarray(x, np.float64)
    return x * (1.0 + eps * rng.uniform(-1.0, 1.0, x.shape))


def rmsnorm(x, g, eps):
    """RMSNorm (Llama/Qwen, SURVEY amb. A13): x / sqrt(mean(x^2) + eps) * g, over the last axis."""
    x = np.asarray(x, np.float64)
    ms = np.mean(x * x, axis=-1, keepdims=True)
    return x / np.sqrt(ms + eps) * g


def rope_angles(pos, head_dim, theta):
    """Rotary angles pos * theta^(-2i/hd), i < hd/2 (SURVEY amb. A14, rotate-half convention)."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    inv_freq = np.power(float(theta), -2.0 * i / head_dim)
    return np.asarray(pos, np.float64)[..., None] * inv_freq


def rope(x, pos, theta):
    """Rotate-half RoPE.  x [..., heads, hd], pos broadcastable to x.shape[:-2].

    out[:h] = x[:h] cos - x[h:] sin ;  out[h:] = x[h:] cos + x[:h] sin   (h = hd/2)
    """
    x = np.asarray(x, np.float64)
    hd = x.shape[-1]
    ang = rope_angles(pos, hd, theta)[..., None, :]        # [..., 1, hd/2]
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(x):
    x = np.asarray(x, np.float64)
    return x / (1.0 + np.exp(-x))


def softmax(s, axis=-1):
    s = np.asarray(s, np.float64)
    m = np.max(s, axis=axis, keepdims=True)
    e = np.exp(s - m)
    return e / np.sum(e, axis=axis, keepdims=True)


# Storage point of the softmax numerator (DESIGN.md R-precision; SURVEY amb. A12: "optionally
# P -> fp16/bf16 to mirror the kernel").  The library's PV product takes P as an fp16 operand
# while the normaliser sums the unrounded exponentials, so the oracle rounds the same point:
# softmax weight = f16(exp(s - max)) / sum exp(s - max).  False = the plain softmax (pins).
ATTN_P_F16 = True


def attention_weights(s):
    """Softmax over the last axis as the PV product consumes it (see ATTN_P_F16); -inf scores
    (masked keys) get weight 0."""
    s = np.asarray(s, np.float64)
    m = np.max(s, axis=-1, keepdims=True)
    e = np.exp(s - m)
    num = f16(perturb(e)) if ATTN_P_F16 else e
    return num / np.sum(e, axis=-1, keepdims=True)


def attention(q, k, v):
    """Scaled-dot-product attention of one query set over one key set (SURVEY amb. A15).

    q [nq, hd], k [nk, hd], v [nk, hd] -> [nq, hd]; scores q.k/sqrt(hd), softmax over keys with
    the numerator stored in fp16 (ATTN_P_F16).
    """
    hd = q.shape[-1]
    s = (q @ k.T) / np.sqrt(hd)
    return attention_weights(s) @ v
