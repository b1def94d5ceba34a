"""Pins of the oracle's numeric building blocks against things other than itself
(SURVEY §8(c) P13): published known-answer vectors, library routines, closed forms."""
import math

import numpy as np
import pytest
import torch

from oracle import philox
from oracle.numerics import bf16, f16, rmsnorm, rope, attention, softmax, silu
from oracle.model import gen_matrix, gen_gain, gen_kv_fill, Weights
from synth.configs import TINY


# Random123 known-answer vectors for philox4x32-10.
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


@pytest.mark.parametrize("ctr,key,expect", KAT)
def test_philox_known_answers(ctr, key, expect):
    out = philox.philox4x32_10(*ctr, *key)
    assert tuple(int(x) for x in out) == expect


def test_philox_words_range_matches_word():
    idx = np.arange(3, 203)
    a = philox.word(idx, 7, 8, 9, 11, 12)
    b = philox.words_range(3, 200, 7, 8, 9, 11, 12)
    assert np.array_equal(a, b)


def test_bf16_matches_torch_rne():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(200000).astype(np.float32),
        (rng.standard_normal(20000) * 1e-30).astype(np.float32),
        (rng.standard_normal(20000) * 1e30).astype(np.float32),
    ])
    # exact ties: values halfway between two bf16 numbers (low 16 bits = 0x8000)
    bits = rng.integers(0, 2**31, 20000, dtype=np.uint32) & np.uint32(0x7FFF0000) | np.uint32(0x8000)
    ties = bits.view(np.float32)
    ties = ties[np.isfinite(ties)]
    x = np.concatenate([x, ties, -ties, np.float32([0.0, -0.0, 1.0, 3.0e38])])
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    got = bf16(x.astype(np.float64))
    assert np.array_equal(got, ref)


def test_f16_matches_numpy_rne():
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.standard_normal(200000) * s for s in (1e-6, 1e-3, 1.0, 1e3, 3e4)])
    # exact ties between fp16 neighbours and subnormals / overflow edges
    h = rng.integers(0, 0x7BFF, 20000).astype(np.uint16).view(np.float16).astype(np.float64)
    h2 = (rng.integers(0, 0x7BFF, 20000).astype(np.uint16) + 1).view(np.float16).astype(np.float64)
    x = np.concatenate([x, (h + h2) / 2, -(h + h2) / 2, [0.0, 65504.0, 65519.0, 65520.0, 2.0 ** -25, 3 * 2.0 ** -26]])
    ref = x.astype(np.float16).astype(np.float64)
    got = f16(x)
    assert np.array_equal(got, ref)


def test_weights_distribution_and_row_slicing():
    d, rows = 256, 512
    w = gen_matrix(3, "wq", 1, rows, d, 1 / math.sqrt(d))
    lim = math.sqrt(3.0 / d)
    assert np.all(np.abs(w) <= lim * 1.004)
    assert abs(w.mean()) < 0.01 * lim
    assert abs(w.var() / (1.0 / d) - 1.0) < 0.02
    # a row generated alone equals the same row of the full matrix (counter = element index)
    assert np.array_equal(gen_matrix(3, "wq", 1, rows, d, 1 / math.sqrt(d), 77, 3), w[77:80])
    # different tensor / layer -> different streams
    assert not np.array_equal(w, gen_matrix(3, "wk", 1, rows, d, 1 / math.sqrt(d)))
    assert not np.array_equal(w, gen_matrix(3, "wq", 0, rows, d, 1 / math.sqrt(d)))
    # all values are bf16-representable
    assert np.array_equal(bf16(w), w)
    g = gen_gain(3, "g_attn", 0, 4096)
    assert np.all((g >= 0.75) & (g <= 1.25)) and g.std() > 0.1


def test_kv_fill_range_and_slicing():
    a = gen_kv_fill(9, 2, 1, 0, 40, 2, 16)
    assert a.shape == (40, 2, 16) and np.all(np.abs(a) <= 1.0)
    b = gen_kv_fill(9, 2, 1, 0, 10, 2, 16, tok_start=30)
    assert np.array_equal(a[30:], b)
    assert not np.array_equal(a, gen_kv_fill(9, 2, 1, 1, 40, 2, 16))


def test_rmsnorm_closed_forms():
    g = np.linspace(0.5, 1.5, 8)
    c = 3.0
    out = rmsnorm(np.full(8, c), g, 1e-6)
    assert np.allclose(out, g * c / math.sqrt(c * c + 1e-6), rtol=1e-15)
    x = np.random.default_rng(1).standard_normal((5, 8))
    assert np.allclose(rmsnorm(7.5 * x, g, 0.0), rmsnorm(x, g, 0.0), rtol=1e-13)
    # unit RMS after normalisation with unit gain
    y = rmsnorm(x, np.ones(8), 0.0)
    assert np.allclose(np.sqrt((y * y).mean(-1)), 1.0)


def test_rope_against_complex_rotation_and_invariants():
    rng = np.random.default_rng(2)
    hd, theta = 16, 10000.0
    x = rng.standard_normal((6, 3, hd))
    pos = np.array([0, 1, 5, 31, 1000, 16383], float)
    out = rope(x, pos, theta)
    # independent formulation: (x1 + i x2) * exp(i * pos * theta^(-2j/hd))
    j = np.arange(hd // 2)
    z = (x[..., : hd // 2] + 1j * x[..., hd // 2:]) * np.exp(
        1j * pos[:, None, None] * theta ** (-2.0 * j / hd))
    assert np.allclose(out[..., : hd // 2], z.real, atol=1e-12)
    assert np.allclose(out[..., hd // 2:], z.imag, atol=1e-12)
    assert np.allclose(out[0], x[0])                      # identity at position 0
    assert np.allclose(np.linalg.norm(out, axis=-1), np.linalg.norm(x, axis=-1))
    # <rope(q, m), rope(k, n)> depends on m - n only
    q, k = rng.standard_normal(hd), rng.standard_normal(hd)
    d1 = rope(q[None, None], np.array([10.0]), theta)[0, 0] @ rope(k[None, None], np.array([3.0]), theta)[0, 0]
    d2 = rope(q[None, None], np.array([107.0]), theta)[0, 0] @ rope(k[None, None], np.array([100.0]), theta)[0, 0]
    assert abs(d1 - d2) < 1e-9


def test_attention_against_torch_sdpa():
    """The plain softmax (ATTN_P_F16 off) is SDPA to fp64 rounding; with the fp16 numerator
    (R-precision) every weight carries one fp16 rounding of relative size <= 2^-11, so
    |o - sdpa| <= 2^-11 * sum_j p_j |v_j| elementwise (p = the exact softmax) — a dropped term,
    a wrong scale or a rounded denominator breaks one of the two."""
    import oracle.numerics as N
    rng = np.random.default_rng(3)
    q, k, v = rng.standard_normal((7, 16)), rng.standard_normal((40, 16)), rng.standard_normal((40, 16))
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q)[None], torch.from_numpy(k)[None], torch.from_numpy(v)[None])[0].numpy()
    N.ATTN_P_F16 = False
    try:
        assert np.allclose(attention(q, k, v), ref, rtol=0, atol=1e-12)
    finally:
        N.ATTN_P_F16 = True
    o = attention(q, k, v)
    p = softmax(q @ k.T / 4.0)
    bound = 2.0 ** -11 * (p @ np.abs(v))
    assert np.all(np.abs(o - ref) <= bound + 1e-12)
    assert np.abs(o - ref).max() > 1e-7          # the rounding is really applied
    # exponentials exactly representable in fp16 (equal scores -> p = 1): no rounding at all
    qz = np.zeros((2, 16))
    assert np.allclose(attention(qz, k, v), v.mean(axis=0)[None].repeat(2, 0), rtol=0, atol=1e-12)
    # the denominator is the unrounded sum: weights of exp values 1 and e^-1 (fp16(e^-1) != e^-1)
    w = N.attention_weights(np.array([[0.0, -1.0]]))
    assert w[0, 0] == 1.0 / (1.0 + np.exp(-1.0)) and w[0, 1] == float(np.float16(np.exp(-1.0))) / (1.0 + np.exp(-1.0))


def test_softmax_silu_closed_forms():
    p = softmax(np.log(np.array([0.8, 0.2])) / 0.5)
    assert np.allclose(p, [0.64 / 0.68, 0.04 / 0.68])   # S:65 example: [0.9412, 0.0588]
    assert np.allclose(silu(np.array([0.0, 1.0])), [0.0, 1.0 / (1.0 + math.exp(-1.0))])


def test_lm_head_blocked_equals_full():
    from oracle.model import lm_logits
    W = Weights(TINY, 5)
    hf = np.random.default_rng(4).standard_normal((3, TINY.d))
    full = hf @ W.lm_head().T
    assert np.allclose(lm_logits(W, hf, block=100, cache_full=False), full, rtol=0, atol=1e-12)
