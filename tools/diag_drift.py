"""Diagnostic: distribution of |logit_gpu - logit_oracle| on the parity-test setup, next to the
noise floor of the oracle itself (same contract, float32 instead of float64 matmuls)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle.model as OM
from oracle import verify as OV
from synth.configs import TINY, TINY_MHA, SMALL128
from synth.trees import pooled_tree
from paper_2505_17052_b200 import api


def stats(d):
    return f"max {d.max():.4f} p99.9 {np.quantile(d, .999):.4f} p99 {np.quantile(d, .99):.4f} mean {d.mean():.5f}"


for shape in (TINY, TINY_MHA, SMALL128):
    rng = np.random.default_rng(202)
    B = 5
    prompts = [[int(t) for t in rng.integers(0, shape.vocab, int(l))] for l in [32, 40, 17, 60, 32]]
    W = OM.Weights(shape, 1)
    model = api.Model(shape, 1, max_position=4096)
    pool = api.KVPool(model, 64, 16)
    ws = model.workspace(B, B * 65, 400)
    ses, hs = [], []
    for i, p in enumerate(prompts):
        ses.append(OV.make_session(W, p, 100 + i))
        h = pool.alloc(400)
        pool.prefill(h, p, ws)
        hs.append(h)
    trees = [pooled_tree(rng, n, 4, 3, shape.vocab) for n in (8, 16, 1, 32, 8)]
    batch = api.Batch.from_host(hs, [s.context_len for s in ses], [s.last_token for s in ses],
                                [s.session_id for s in ses], [0] * B, trees, max_context_len=400)
    out = api.verify(model, pool, batch, ws, auto_commit=False)
    lg = api.debug_last_logits(model, ws, batch).cpu().numpy()
    refs = OV.verify_batch(W, [OV.Request(s, t.parent, t.token) for s, t in zip(ses, trees)], auto_commit=False)
    ref = np.concatenate([o.logits for o in refs])
    print(shape.name, "gpu vs oracle:", stats(np.abs(lg - ref)), "logit std", ref.std().round(3))
    # oracle noise floor: same storage contract, float32 matmuls
    mm = np.ndarray.__matmul__
    orig = OM._qkv, OM._post_attn
    def f32mm(a, b):
        return (a.astype(np.float32) @ b.astype(np.float32)).astype(np.float64)
    def qkv(Wt, l, x, pos):
        s = Wt.shape; Lw = Wt.layer(l)
        h = OM.bf16(OM.rmsnorm(x, Lw["g_attn"], s.eps))
        q = f32mm(h, Lw["wq"].T).reshape(-1, s.n_heads, s.head_dim)
        k = f32mm(h, Lw["wk"].T).reshape(-1, s.n_kv, s.head_dim)
        v = f32mm(h, Lw["wv"].T).reshape(-1, s.n_kv, s.head_dim)
        return OM.bf16(OM.rope(q, pos, s.rope_theta)), OM.bf16(OM.rope(k, pos, s.rope_theta)), OM.bf16(v)
    def post(Wt, l, x, o):
        s = Wt.shape; Lw = Wt.layer(l)
        O = OM.bf16(o.reshape(o.shape[0], -1)); x = x + f32mm(O, Lw["wo"].T)
        h2 = OM.bf16(OM.rmsnorm(x, Lw["g_mlp"], s.eps))
        M = OM.bf16(OM.silu(f32mm(h2, Lw["wg"].T)) * f32mm(h2, Lw["wu"].T))
        return x + f32mm(M, Lw["wd"].T)
    OM._qkv, OM._post_attn = qkv, post
    try:
        ses2 = [OV.make_session(W, p, 100 + i) for i, p in enumerate(prompts)]
        refs2 = OV.verify_batch(W, [OV.Request(s, t.parent, t.token) for s, t in zip(ses2, trees)], auto_commit=False)
    finally:
        OM._qkv, OM._post_attn = orig
    ref2 = np.concatenate([o.logits for o in refs2])
    print(shape.name, "oracle f32-matmul vs f64:", stats(np.abs(ref2 - ref)))
    pool.close(); model.close()
