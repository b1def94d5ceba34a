"""Kernel-level parity on a B200: weights (bit-exact), tcgen05 GEMM, tree attention.
All calls go through libspecedge's C ABI."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.model import gen_matrix, gen_gain, Weights  # noqa: E402
from oracle.numerics import attention, bf16, f16  # noqa: E402
from synth.configs import TINY, LLAMA3_8B_2L, SMALL128  # noqa: E402
from tests.gpu_helpers import ATTN_TOL, bf16_bits_to_f64  # noqa: E402


@pytest.fixture(scope="module")
def api():
    from paper_2505_17052_b200 import api as A
    return A


def _rand_bf16(rng, shape, scale=1.0):
    x = bf16(rng.standard_normal(shape) * scale).astype(np.float32)
    return torch.from_numpy(x).to(torch.bfloat16).cuda()


def _rand_f16(rng, shape, scale=1.0):
    x = f16(rng.standard_normal(shape) * scale).astype(np.float32)
    return torch.from_numpy(x).to(torch.float16).cuda()


# ------------------------------------------------------------------ K12: bit-identical weights
TENSORS = [(1, "embed", None), (2, "wq", "q"), (3, "wk", "k"), (4, "wv", "k"), (5, "wo", "o"), (6, "wg", "f"),
           (7, "wu", "f"), (8, "wd", "d"), (9, "lm_head", None), (10, "g_attn", "g"), (11, "g_mlp", "g"),
           (12, "g_final", "g")]


def _oracle_rows(shape, seed, name, layer, rows):
    s = shape
    qd, kd = s.n_heads * s.head_dim, s.n_kv * s.head_dim
    if name.startswith("g_"):
        return gen_gain(seed, name, layer, s.d)[None]
    dims = dict(embed=(s.vocab, s.d, 1.0), wq=(qd, s.d, 1 / math.sqrt(s.d)), wk=(kd, s.d, 1 / math.sqrt(s.d)),
                wv=(kd, s.d, 1 / math.sqrt(s.d)), wo=(s.d, qd, 1 / math.sqrt(qd)),
                wg=(s.ffn, s.d, 1 / math.sqrt(s.d)), wu=(s.ffn, s.d, 1 / math.sqrt(s.d)),
                wd=(s.d, s.ffn, 1 / math.sqrt(s.ffn)), lm_head=(s.vocab, s.d, 2 / math.sqrt(s.d)))[name]
    return np.concatenate([gen_matrix(seed, name, layer, dims[0], dims[1], dims[2], r, 1) for r in rows])


@pytest.mark.parametrize("shape", [TINY, LLAMA3_8B_2L])
def test_weights_bit_identical_to_oracle(api, shape):
    m = api.Model(shape, 77, max_position=4096)
    rng = np.random.default_rng(0)
    try:
        for tid, name, kind in TENSORS:
            layers = [0] if name in ("embed", "lm_head", "g_final") else list(range(shape.n_layers))
            for layer in layers:
                s = shape
                nrows = dict(q=s.n_heads * s.head_dim, k=s.n_kv * s.head_dim, o=s.d, f=s.ffn, d=s.d, g=1).get(
                    kind, s.vocab)
                cols = dict(o=s.n_heads * s.head_dim, d=s.ffn).get(kind, s.d)
                rows = list(range(nrows)) if nrows <= 512 else sorted(set(
                    [0, 1, 63, 64, 127, 128, nrows - 1] + list(rng.integers(0, nrows, 8))))
                ref = _oracle_rows(shape, 77, name, layer, rows)
                got = np.concatenate([m.weight_rows(tid, layer, r, 1, cols) for r in rows])
                assert np.array_equal(bf16_bits_to_f64(got), ref), (name, layer)
    finally:
        m.close()


# ------------------------------------------------------------------ tcgen05 GEMM
@pytest.mark.parametrize("M,R,K", [(128, 9, 64), (256, 33, 128), (200, 100, 192), (384, 257, 256),
                                   (1024, 528, 4096), (128, 16, 14336), (640, 1056, 512)])
def test_gemm_matches_fp64(api, M, R, K):
    rng = np.random.default_rng(M * 7 + R)
    W = _rand_bf16(rng, (M, K), 1 / math.sqrt(K))
    X = _rand_bf16(rng, (R, K))
    out = api.debug_gemm(W, X).cpu().numpy().astype(np.float64)
    ref = X.float().cpu().double().numpy() @ W.float().cpu().double().numpy().T
    err = np.abs(out - ref)
    assert err.max() <= 1e-3 * max(1.0, np.abs(ref).max()), err.max()


# ------------------------------------------------------------------ tree attention
def _anc_masks(parent):
    anc = []
    for i, p in enumerate(parent):
        anc.append((0 if p < 0 else anc[p]) | (1 << i))
    return anc


# tcgen05 kernel (hd 64/128) pass structure (attention_tc.cu): (128,4,1000,32,*) pair pass with a
# 4-row tail replicated x4; (128,5,300,32,1) pair pass, 40-row tail replicated x2; (128,8,4097,64,8)
# two pair passes + a single pass whose 8-row tile is replicated x4 (8 partials merged);
# (128,4,500,11,1) single pass replicated x2; (128,4,700,5,2) single pass replicated x4;
# (128,5,64,16,1) / (128,4,0,20,1) single pass without replication (2 in-CTA KV streams).
@pytest.mark.parametrize("hd,G,L,N,splits", [(16, 2, 31, 8, 1), (128, 4, 1000, 32, 4), (128, 5, 64, 16, 1),
                                             (64, 8, 200, 64, 3), (128, 4, 0, 20, 1), (32, 1, 130, 0, 2),
                                             (128, 8, 4097, 64, 8), (128, 4, 1000, 32, 1), (128, 5, 300, 32, 1),
                                             (128, 4, 500, 11, 1), (128, 4, 700, 5, 2), (64, 4, 333, 32, 1)])
def test_tree_attention_matches_oracle(api, hd, G, L, N, splits):
    from synth.trees import random_tree
    rng = np.random.default_rng(hd + G + L + N)
    S = N + 1
    tree = random_tree(rng, N, 1000)
    q = _rand_f16(rng, (S, G, hd))          # attention operands are fp16 (DESIGN R-precision)
    kp = _rand_f16(rng, (max(L, 1), hd))[:L] if L else None
    vp = _rand_f16(rng, (max(L, 1), hd))[:L] if L else None
    kt = _rand_f16(rng, (S, hd))
    vt = _rand_f16(rng, (S, hd))
    anc = np.array(_anc_masks(tree.parent), dtype=np.uint64).view(np.int64)
    anc_t = torch.from_numpy(anc).cuda() if N else torch.zeros(1, dtype=torch.int64, device="cuda")
    o = api.debug_attention(q, kp, vp, kt, vt, anc_t, n_splits=splits).cpu().numpy().astype(np.float64)
    qn = q.float().cpu().double().numpy()
    kpn = kp.float().cpu().double().numpy() if L else np.zeros((0, hd))
    vpn = vp.float().cpu().double().numpy() if L else np.zeros((0, hd))
    ktn, vtn = kt.float().cpu().double().numpy(), vt.float().cpu().double().numpy()
    vis = [[0]]
    for i, p in enumerate(tree.parent):
        vis.append((vis[0] if p < 0 else vis[p + 1]) + [i + 1])
    worst = 0.0
    for s in range(S):
        keys = np.concatenate([kpn, ktn[vis[s]]])
        vals = np.concatenate([vpn, vtn[vis[s]]])
        for j in range(G):
            ref = attention(qn[s, j][None], keys, vals)[0]
            rel = np.linalg.norm(o[s, j] - ref) / max(np.linalg.norm(ref), 1e-30)
            worst = max(worst, rel)
    assert worst <= ATTN_TOL, worst


@pytest.mark.parametrize("hd,G,L,N,splits", [(128, 4, 2000, 32, 1), (128, 5, 3000, 16, 4), (128, 8, 4000, 64, 2),
                                             (64, 4, 1500, 20, 1)])
def test_tree_attention_rescale_heavy(api, hd, G, L, N, splits):
    """Scores whose scale grows along the context, differently per query row: the running max
    keeps rising, so lanes of one warp disagree on the lazy O rescale (the case that once hung a
    warp on its warp-collective TMEM loads).  Same fp64 reference as above."""
    from synth.trees import random_tree
    rng = np.random.default_rng(7 * hd + G + L + N)
    S = N + 1
    tree = random_tree(rng, N, 1000)
    qf = rng.standard_normal((S, G, hd)) * (1.0 + 3.0 * rng.random((S, G, 1)))
    ramp = (1.0 + 5.0 * np.arange(L) / max(L, 1))[:, None]
    kf = rng.standard_normal((L, hd)) * ramp
    q = torch.from_numpy(qf.astype(np.float16)).cuda()
    kp = torch.from_numpy(kf.astype(np.float16)).cuda()
    vp = _rand_f16(rng, (L, hd))
    kt = torch.from_numpy((rng.standard_normal((S, hd)) * 6.0).astype(np.float16)).cuda()
    vt = _rand_f16(rng, (S, hd))
    anc = np.array(_anc_masks(tree.parent), dtype=np.uint64).view(np.int64)
    anc_t = torch.from_numpy(anc).cuda()
    o = api.debug_attention(q, kp, vp, kt, vt, anc_t, n_splits=splits).cpu().numpy().astype(np.float64)
    qn = q.float().cpu().double().numpy()
    kpn, vpn = kp.float().cpu().double().numpy(), vp.float().cpu().double().numpy()
    ktn, vtn = kt.float().cpu().double().numpy(), vt.float().cpu().double().numpy()
    vis = [[0]]
    for i, p in enumerate(tree.parent):
        vis.append((vis[0] if p < 0 else vis[p + 1]) + [i + 1])
    worst = 0.0
    for s in range(S):
        keys = np.concatenate([kpn, ktn[vis[s]]])
        vals = np.concatenate([vpn, vtn[vis[s]]])
        for j in range(G):
            ref = attention(qn[s, j][None], keys, vals)[0]
            rel = np.linalg.norm(o[s, j] - ref) / max(np.linalg.norm(ref), 1e-30)
            worst = max(worst, rel)
    assert worst <= ATTN_TOL, worst
