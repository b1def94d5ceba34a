"""External pin of the oracle's decoder-layer composition (oracle/model.py _qkv / _post_attn:
RMSNorm gain placement, rotate-half RoPE, GQA head -> kv-head map, softmax scale, O-proj and MLP
residual points, silu(gate) * up): with its storage roundings switched off, one oracle layer over a
causal chain equals the Hugging Face transformers LlamaDecoderLayer (SURVEY amb. A13-A16 name the
Llama/Qwen3 layout) carrying the same Philox weights, in float64."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

import oracle.model as OM  # noqa: E402
import oracle.numerics as ON  # noqa: E402
from synth.configs import ModelShape  # noqa: E402

SHAPE = ModelShape("hf-pin", 1, 128, 4, 2, 32, 256, 64, 1e-5, 10000.0)


def _hf_layer(W):
    from transformers.models.llama import modeling_llama as M
    s = W.shape
    cfg = transformers.LlamaConfig(hidden_size=s.d, intermediate_size=s.ffn, num_attention_heads=s.n_heads,
                                   num_key_value_heads=s.n_kv, head_dim=s.head_dim, rms_norm_eps=s.eps,
                                   max_position_embeddings=256, vocab_size=s.vocab, attention_bias=False,
                                   mlp_bias=False, hidden_act="silu")
    cfg.rope_theta = s.rope_theta
    if getattr(cfg, "rope_parameters", None) is not None:
        cfg.rope_parameters = {"rope_type": "default", "rope_theta": s.rope_theta}
    cfg._attn_implementation = "eager"
    layer = M.LlamaDecoderLayer(cfg, 0).double()
    rot = M.LlamaRotaryEmbedding(cfg)
    Lw = W.layer(0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64))
    with torch.no_grad():
        layer.self_attn.q_proj.weight.copy_(t(Lw["wq"]))
        layer.self_attn.k_proj.weight.copy_(t(Lw["wk"]))
        layer.self_attn.v_proj.weight.copy_(t(Lw["wv"]))
        layer.self_attn.o_proj.weight.copy_(t(Lw["wo"]))
        layer.mlp.gate_proj.weight.copy_(t(Lw["wg"]))
        layer.mlp.up_proj.weight.copy_(t(Lw["wu"]))
        layer.mlp.down_proj.weight.copy_(t(Lw["wd"]))
        layer.input_layernorm.weight.copy_(t(Lw["g_attn"]))
        layer.post_attention_layernorm.weight.copy_(t(Lw["g_mlp"]))
    return layer, rot


def _oracle_layer_unrounded(W, x):
    """One oracle layer (the composition tree_forward / decode / prefill_dense use) over a causal
    chain at positions 0..n-1, storage roundings off."""
    s = W.shape
    n = x.shape[0]
    pos = np.arange(n, dtype=np.float64)
    ident = lambda a: np.asarray(a, np.float64)
    saved = (OM.bf16, OM.f16, ON.ATTN_P_F16)
    OM.bf16, OM.f16, ON.ATTN_P_F16 = ident, ident, False
    try:
        q, k, v = OM._qkv(W, 0, x, pos)
        o = np.empty_like(q)
        mask = np.tril(np.ones((n, n), bool))
        for h in range(s.n_heads):
            g = h // s.group
            sc = (q[:, h] @ k[:, g].T) / np.sqrt(s.head_dim)
            o[:, h] = ON.attention_weights(np.where(mask, sc, -np.inf)) @ v[:, g]
        return OM._post_attn(W, 0, x, o)
    finally:
        OM.bf16, OM.f16, ON.ATTN_P_F16 = saved


def test_oracle_layer_equals_hf_llama_decoder_layer():
    W = OM.Weights(SHAPE, 21)
    layer, rot = _hf_layer(W)
    rng = np.random.default_rng(3)
    n = 11
    x = rng.standard_normal((n, SHAPE.d))
    ours = _oracle_layer_unrounded(W, x)
    xt = torch.from_numpy(x)[None]
    pid = torch.arange(n)[None]
    mask = torch.full((n, n), float("-inf"), dtype=torch.float64).triu(1)[None, None]

    def hf(cos, sin):
        with torch.no_grad():
            out = layer(xt, attention_mask=mask, position_ids=pid, position_embeddings=(cos, sin))
        return (out[0] if isinstance(out, tuple) else out)[0].numpy()
    # RoPE tables in float64 (amb. A14: angles in double), in HF's duplicated-half layout
    ang = ON.rope_angles(np.arange(n, dtype=np.float64), SHAPE.head_dim, SHAPE.rope_theta)
    c = torch.from_numpy(np.concatenate([np.cos(ang), np.cos(ang)], -1))[None]
    sn = torch.from_numpy(np.concatenate([np.sin(ang), np.sin(ang)], -1))[None]
    out = hf(c, sn)
    # HF's LlamaRMSNorm evaluates in float32 (x.to(float32) * rsqrt(mean x^2 + eps)): agreement to
    # float32 rounding (~1e-7 relative); a composition error (gain, residual point, head map, gate/up)
    # is O(1)
    assert np.abs(out - ours).max() <= 2e-6 * max(1.0, np.abs(ours).max()), np.abs(out - ours).max()
    # HF's own rotary embedding (float32 inverse frequencies) gives the same to ~1e-6
    cos32, sin32 = rot(xt, pid)
    assert np.abs(hf(cos32.double(), sin32.double()) - ours).max() <= 1e-5
    # and it is a real check: a dropped gain or a swapped gate/up breaks it
    Lw = W.layer(0)
    Lw["wg"], Lw["wu"] = Lw["wu"], Lw["wg"]
    assert np.abs(_oracle_layer_unrounded(W, x) - out).max() > 1e-3
