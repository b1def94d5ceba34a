"""Target decoder of the verifier, float64 with bf16 storage points.

The paper runs "the server model" over all draft tokens "in a single forward pass" (P:171,
§4.1) with a per-sequence custom attention mask (§4.3); it never names the
architecture's details beyond the target families (Qwen3 / Llama / Vicuna).  The
decoder here is the Llama/Qwen3 family layout (SURVEY amb. A13-A16): RMSNorm -> QKV -> RoPE ->
GQA attention -> O-proj + residual -> RMSNorm -> SwiGLU MLP + residual, final RMSNorm, untied
LM head, no biases, QK-norm off.

Storage points (reading R-precision, revising SURVEY amb. A12): bf16 for weights,
embeddings and the GEMM input operands (normed h, attention output O, MLP hidden M); fp16 for the
attention operands q, k (post-RoPE) and v, hence the KV cache, and for the softmax numerator P
as the PV product consumes it (numerics.attention_weights; P in bf16 would break the 1e-3
attention tolerance).  Unrounded: the residual stream
x (the GPU keeps it in fp32) and the final-norm output (the GPU passes it to the LM head as a
hi/lo pair of bf16 operands); rounding those two amplifies arithmetic-order noise past the
north_star logit tolerance (measured).

Two independent ways of running it live here:
  * `tree_forward`   - SURVEY §8(c) O2: all S = N+1 slots of a draft tree at once; slot s
                       attends to the cached prefix, the root and its own ancestors-or-self;
  * `decode`         - SURVEY §8(c) O6: the plain definition, one token at a time with an
                       ordinary causal KV cache (textbook autoregressive decoding);
  * `prefill_dense`  - textbook causal attention of a whole sequence with a causal mask.
Tests pin tree_forward == decode along every root-to-node path (P1) and chain == prefill (P2).

Weights: every element is
    bf16( f32( f32(int24) * scale_t ) ),  int24 = (x >> 8) - 2^23,
x = Philox4x32-10 word (key = seed split lo/hi, counter = (idx>>2, tensor_id, layer, 'WEIG'),
word idx & 3), idx = row * cols + col of the logical row-major matrix.  scale_t =
f32(std_t * sqrt(3) * 2^-23) so that values are U(-sqrt(3) std, sqrt(3) std).  std: embedding
1, projections 1/sqrt(fan_in), LM head 2/sqrt(d) (logit std ~ 2).  Norm gains are
bf16(f32(f32(int24) * 2^-25) + 1) in [0.75, 1.25) (random so that a dropped gain is caught).
"""
from __future__ import annotations

import math

import numpy as np

from . import philox
from .numerics import bf16, f16, rmsnorm, rope, silu, attention, attention_weights, perturb

# Matmul arithmetic of the oracle.  float64 is the reference; tests switch it to float32 (same
# storage contract) to measure the oracle's own arithmetic-noise floor, against which the
# library's floating-point agreement is calibrated.
MATMUL_DTYPE = np.float64


def _mm(a, b):
    if MATMUL_DTYPE == np.float64:
        return a @ b
    return (a.astype(MATMUL_DTYPE) @ b.astype(MATMUL_DTYPE)).astype(np.float64)


TENSOR_ID = dict(embed=1, wq=2, wk=3, wv=4, wo=5, wg=6, wu=7, wd=8, lm_head=9,
                 g_attn=10, g_mlp=11, g_final=12)
WEIGHT_TAG = 0x57454947  # 'WEIG'
KVFILL_TAG = 0x4B564649  # 'KVFI'


def _int24(words):
    return (words >> np.uint64(8)).astype(np.int64) - (1 << 23)


def gen_matrix(seed, tensor, layer, rows, cols, std, row_start=0, row_count=None):
    """Rows [row_start, row_start+row_count) of the logical [rows, cols] weight (O1)."""
    if row_count is None:
        row_count = rows - row_start
    k0, k1 = philox.split_seed(seed)
    w = philox.words_range(row_start * cols, row_count * cols, TENSOR_ID[tensor], layer,
                           WEIGHT_TAG, k0, k1)
    scale = np.float32(std * math.sqrt(3.0) * 2.0 ** -23)
    v = _int24(w).astype(np.float32) * scale          # one IEEE fp32 rounding
    return bf16(v.astype(np.float64)).reshape(row_count, cols)


def gen_gain(seed, tensor, layer, d):
    k0, k1 = philox.split_seed(seed)
    w = philox.words_range(0, d, TENSOR_ID[tensor], layer, WEIGHT_TAG, k0, k1)
    v = _int24(w).astype(np.float32) * np.float32(2.0 ** -25) + np.float32(1.0)
    return bf16(v.astype(np.float64))


def gen_kv_fill(seed, stream, layer, kv_sel, n_tok, n_kv, hd, tok_start=0):
    """Synthetic cached K or V rows (perf runs fill the prefix instead of
    prefilling).  Element e = head*hd + j of token position t is f16(f32(int24 * 2^-23)) in
    [-1, 1) from Philox counter (e >> 2, t, layer*2 + kv_sel, stream ^ 'KVFI'), word e & 3.
    Returns [n_tok, n_kv, hd]."""
    k0, k1 = philox.split_seed(seed)
    per_tok = n_kv * hd
    assert per_tok % 4 == 0
    c0 = np.arange(per_tok // 4, dtype=np.uint64)[None, :]
    c1 = np.arange(tok_start, tok_start + n_tok, dtype=np.uint64)[:, None]
    r = philox.philox4x32_10(c0, c1, (layer << 1) | kv_sel, stream ^ KVFILL_TAG, k0, k1)
    w = np.stack(r, axis=-1).reshape(n_tok, per_tok)
    v = _int24(w).astype(np.float32) * np.float32(2.0 ** -23)
    return f16(v.astype(np.float64)).reshape(n_tok, n_kv, hd)


class Weights:
    """Lazily generated logical weights of one model (float64 arrays of bf16 values)."""

    def __init__(self, shape, seed):
        self.shape = shape
        self.seed = seed
        self._layers = {}
        self._lm = None
        self._g_final = None

    def embed_rows(self, tokens):
        s = self.shape
        rows = [gen_matrix(self.seed, "embed", 0, s.vocab, s.d, 1.0, int(t), 1)[0] for t in tokens]
        return np.stack(rows) if rows else np.zeros((0, s.d))

    def layer(self, l):
        if l not in self._layers:
            s = self.shape
            qd, kd = s.n_heads * s.head_dim, s.n_kv * s.head_dim
            self._layers[l] = dict(
                wq=gen_matrix(self.seed, "wq", l, qd, s.d, 1 / math.sqrt(s.d)),
                wk=gen_matrix(self.seed, "wk", l, kd, s.d, 1 / math.sqrt(s.d)),
                wv=gen_matrix(self.seed, "wv", l, kd, s.d, 1 / math.sqrt(s.d)),
                wo=gen_matrix(self.seed, "wo", l, s.d, qd, 1 / math.sqrt(qd)),
                wg=gen_matrix(self.seed, "wg", l, s.ffn, s.d, 1 / math.sqrt(s.d)),
                wu=gen_matrix(self.seed, "wu", l, s.ffn, s.d, 1 / math.sqrt(s.d)),
                wd=gen_matrix(self.seed, "wd", l, s.d, s.ffn, 1 / math.sqrt(s.ffn)),
                g_attn=gen_gain(self.seed, "g_attn", l, s.d),
                g_mlp=gen_gain(self.seed, "g_mlp", l, s.d),
            )
        return self._layers[l]

    def drop_layer(self, l):
        self._layers.pop(l, None)

    def g_final(self):
        if self._g_final is None:
            self._g_final = gen_gain(self.seed, "g_final", 0, self.shape.d)
        return self._g_final

    def lm_head_block(self, v0, nv):
        s = self.shape
        return gen_matrix(self.seed, "lm_head", 0, s.vocab, s.d, 2 / math.sqrt(s.d), v0, nv)

    def lm_head(self):
        if self._lm is None:
            self._lm = self.lm_head_block(0, self.shape.vocab)
        return self._lm


def lm_logits(W: Weights, hf, block=16384, cache_full=True):
    """logits = hf . Wlm^T (float64, never rounded; SURVEY §8(c) O2 last line)."""
    s = W.shape
    if cache_full and s.vocab <= 65536:
        return _mm(hf, W.lm_head().T)
    out = np.empty((hf.shape[0], s.vocab))
    for v0 in range(0, s.vocab, block):
        nv = min(block, s.vocab - v0)
        out[:, v0:v0 + nv] = _mm(hf, W.lm_head_block(v0, nv).T)
    return out


# ----------------------------------------------------------------------------------------------
# KV cache: per layer, K and V arrays [L, n_kv, hd] of fp16 values (post-RoPE K).
# ----------------------------------------------------------------------------------------------
class Cache:
    def __init__(self, shape):
        self.shape = shape
        self.k = [np.zeros((0, shape.n_kv, shape.head_dim)) for _ in range(shape.n_layers)]
        self.v = [np.zeros((0, shape.n_kv, shape.head_dim)) for _ in range(shape.n_layers)]

    def __len__(self):
        return self.k[0].shape[0]

    def copy(self):
        c = Cache(self.shape)
        c.k = [a.copy() for a in self.k]
        c.v = [a.copy() for a in self.v]
        return c

    def append(self, l, k, v):
        self.k[l] = np.concatenate([self.k[l], k], axis=0)
        self.v[l] = np.concatenate([self.v[l], v], axis=0)


def _qkv(W: Weights, l, x, pos):
    s = W.shape
    Lw = W.layer(l)
    h = bf16(perturb(rmsnorm(x, Lw["g_attn"], s.eps)))
    q = _mm(h, Lw["wq"].T).reshape(-1, s.n_heads, s.head_dim)
    k = _mm(h, Lw["wk"].T).reshape(-1, s.n_kv, s.head_dim)
    v = _mm(h, Lw["wv"].T).reshape(-1, s.n_kv, s.head_dim)
    q = f16(perturb(rope(q, pos, s.rope_theta)))
    k = f16(perturb(rope(k, pos, s.rope_theta)))
    return q, k, f16(perturb(v))


def _post_attn(W: Weights, l, x, o):
    """o [n, H, hd] fp64 attention output -> residual stream after the MLP."""
    s = W.shape
    Lw = W.layer(l)
    O = bf16(perturb(o.reshape(o.shape[0], -1)))
    x = x + _mm(O, Lw["wo"].T)             # residual stream is not a GEMM operand: not rounded
    h2 = bf16(perturb(rmsnorm(x, Lw["g_mlp"], s.eps)))
    M = bf16(perturb(silu(_mm(h2, Lw["wg"].T)) * _mm(h2, Lw["wu"].T)))
    return x + _mm(M, Lw["wd"].T)


def final_hidden(W: Weights, x):
    """Final RMSNorm output.  Not rounded: the library feeds it to the LM head as a hi/lo pair of
    bf16 operands (hi + lo = value to ~2^-17 relative), reading R-precision."""
    return rmsnorm(x, W.g_final(), W.shape.eps)


def tree_depth(parent):
    d = np.zeros(len(parent), np.int64)
    for i, p in enumerate(parent):
        d[i] = 1 if p < 0 else d[p] + 1
    return d


def visible_slots(parent):
    """For every slot s (0 = root, i+1 = node i): the tree slots it attends to, ascending —
    the root plus its ancestors-or-self (SURVEY amb. A4; P:316 'custom attention masking for each
    token sequence')."""
    vis = [[0]]
    for i, p in enumerate(parent):
        base = vis[0] if p < 0 else vis[p + 1]
        vis.append(base + [i + 1])
    return vis


def tree_forward(W: Weights, cache: Cache, root_token, parent, token, want_hidden=False):
    """SURVEY §8(c) O2.  Slot 0 = the root (last committed token) at position L = len(cache)
    (amb. A2); node i at position L + depth(i) (amb. A3).  Returns (hf [S, d], tree K/V per layer)
    where tree K/V are lists of [S, n_kv, hd]."""
    s = W.shape
    L = len(cache)
    toks = [int(root_token)] + [int(t) for t in token]
    pos = np.concatenate([[L], L + tree_depth(parent)]).astype(np.float64)
    vis = visible_slots(parent)
    x = W.embed_rows(toks)
    tk, tv = [], []
    G = s.group
    for l in range(s.n_layers):
        q, k, v = _qkv(W, l, x, pos)
        tk.append(k)
        tv.append(v)
        o = np.empty_like(q)
        for si in range(len(toks)):
            keys = np.concatenate([cache.k[l], k[vis[si]]], axis=0)
            vals = np.concatenate([cache.v[l], v[vis[si]]], axis=0)
            for h in range(s.n_heads):
                o[si, h] = attention(q[si, h][None], keys[:, h // G], vals[:, h // G])[0]
        x = _post_attn(W, l, x, o)
    hf = final_hidden(W, x)
    return hf, tk, tv


def decode(W: Weights, cache: Cache, tokens):
    """SURVEY §8(c) O6, the plain definition: feed `tokens` one at a time at positions
    len(cache), len(cache)+1, ...; each attends to every cached position and itself.  Appends
    K/V to `cache` (in place) and returns hf [n, d] (final-norm hidden per step)."""
    s = W.shape
    G = s.group
    outs = []
    for t in tokens:
        pos = np.array([float(len(cache))])
        x = W.embed_rows([int(t)])
        for l in range(s.n_layers):
            q, k, v = _qkv(W, l, x, pos)
            cache.append(l, k, v)
            o = np.empty_like(q)
            for h in range(s.n_heads):
                o[0, h] = attention(q[0, h][None], cache.k[l][:, h // G], cache.v[l][:, h // G])[0]
            x = _post_attn(W, l, x, o)
        outs.append(final_hidden(W, x)[0])
    return np.stack(outs) if outs else np.zeros((0, s.d))


def prefill_dense(W: Weights, tokens):
    """Textbook causal self-attention of a whole sequence at once (explicit lower-triangular
    mask), positions 0..n-1.  Returns (hf [n, d], Cache)."""
    s = W.shape
    G = s.group
    n = len(tokens)
    pos = np.arange(n, dtype=np.float64)
    x = W.embed_rows(tokens)
    cache = Cache(s)
    mask = np.tril(np.ones((n, n), bool))
    for l in range(s.n_layers):
        q, k, v = _qkv(W, l, x, pos)
        cache.append(l, k, v)
        o = np.empty_like(q)
        for h in range(s.n_heads):
            sc = (q[:, h] @ k[:, h // G].T) / np.sqrt(s.head_dim)
            sc = np.where(mask, sc, -np.inf)
            o[:, h] = attention_weights(sc) @ v[:, h // G]
        x = _post_attn(W, l, x, o)
    return final_hidden(W, x), cache
