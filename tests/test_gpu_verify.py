"""End-to-end parity of specedge_verify_batch (through the C ABI) against the oracle on the same
seeded inputs (SURVEY §8(c) tolerances, amb. A21; the contract is spelled out in
tests/gpu_helpers.py):
  - target token per slot: exact where the oracle margin exceeds 1e-2;
  - accept walk + bonus: exact on the library's own targets, always; equal to the oracle's
    outcome unless the first divergent visited slot has oracle margin <= 1e-2 (exempt, counted);
  - committed KV: bit-exact indices (pages == tree-scratch rows of the accepted slots);
  - logits: max-abs <= 2e-2, or 1.25 x the oracle's own float32-vs-float64 deviation where that
    is larger, and 99.9 % within 2e-2 (fp32 capture of the same LM-head kernel);
  - stochastic mode: the (stop node, bonus) law passes chi-square against the oracle's closed
    form (O7) on V = 16.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import verify as OV  # noqa: E402
from oracle.law import closed_form_law, slot_probs  # noqa: E402
from oracle.model import Weights, Cache, gen_kv_fill, lm_logits, tree_forward  # noqa: E402
from synth.configs import TINY, TINY_V16, TINY_MHA, SMALL128, LLAMA3_8B_2L, QWEN3_14B_2L, ModelShape  # noqa: E402
from synth.plant import plant, draw_accept_lengths  # noqa: E402
from synth.trees import pooled_tree, random_tree, chain_tree, Tree  # noqa: E402
from tests.gpu_helpers import (f16_bits_to_f64, check_request, check_batch, check_commit,  # noqa: E402
                               split_outputs, oracle_noise_floor, check_logits, logit_bound)


@pytest.fixture(scope="module")
def api():
    from paper_2505_17052_b200 import api as A
    return A


class Pair:
    """The same sessions on both sides: oracle Sessions and library KV handles."""

    def __init__(self, api, shape, seed, prompts, session_ids, max_nodes=64, capacity=None, num_pages=None,
                 max_requests=None):
        self.api, self.shape = api, shape
        self.W = Weights(shape, seed)
        self.model = api.Model(shape, seed, max_position=4096)
        cap = capacity or max(len(p) for p in prompts) + 256
        pages_per = (cap + 63) // 64
        self.pool = api.KVPool(self.model, num_pages or pages_per * len(prompts) + 4, len(prompts) + 4)
        B = max_requests or len(prompts)
        self.ws = self.model.workspace(B, B * (max_nodes + 1), cap)
        self.sessions, self.handles = [], []
        for p, sid in zip(prompts, session_ids):
            self.sessions.append(OV.make_session(self.W, p, sid))
            h = self.pool.alloc(cap)
            self.pool.prefill(h, p, self.ws)
            self.handles.append(h)
        torch.cuda.synchronize()

    def close(self):
        self.pool.close()
        self.model.close()

    def oracle_targets(self, idx):
        def targets(trees):
            return [OV.verify_one(self.W, OV.Request(self.sessions[i], t.parent, t.token), keep_logits=False).row_target
                    for i, t in zip(idx, trees)]
        return targets

    def batch(self, idx, trees, rounds=None, max_nodes=None):
        api = self.api
        ses = [self.sessions[i] for i in idx]
        return api.Batch.from_host([self.handles[i] for i in idx], [s.context_len for s in ses],
                                   [s.last_token for s in ses], [s.session_id for s in ses],
                                   rounds if rounds is not None else [s.round for s in ses], trees,
                                   max_context_len=max(s.context_len for s in ses) + 8, max_nodes=max_nodes)


def _prompts(rng, n, lens, vocab):
    return [[int(t) for t in rng.integers(0, vocab, int(l))] for l in lens[:n]]


def test_library_prefill_matches_oracle_cache(api):
    rng = np.random.default_rng(101)
    prompts = _prompts(rng, 3, [32, 70, 5], TINY.vocab)    # 70 -> two prefill chunks
    pr = Pair(api, TINY, 1, prompts, [11, 12, 13])
    try:
        assert list(pr.pool.get_len(pr.handles)) == [31, 69, 4]
        for i, s in enumerate(pr.sessions):
            for l in range(TINY.n_layers):
                for kv_sel, ref in ((0, s.cache.k[l]), (1, s.cache.v[l])):
                    got = f16_bits_to_f64(pr.pool.read_kv(pr.handles[i], l, kv_sel, 0, len(s.cache)))
                    # fp16 storage of values computed through bf16 GEMM operands: per cached vector the
                    # norm-wise relative error stays at the 16-bit rounding level
                    num = np.linalg.norm((got - ref).reshape(len(s.cache), -1), axis=1)
                    den = np.linalg.norm(ref.reshape(len(s.cache), -1), axis=1)
                    assert (num / np.maximum(den, 1e-30)).max() <= 2e-2, (i, l, kv_sel)
    finally:
        pr.close()


@pytest.mark.parametrize("shape", [TINY, TINY_MHA, SMALL128])
def test_verify_greedy_matches_oracle(api, shape):
    rng = np.random.default_rng(202)
    B = 5
    prompts = _prompts(rng, B, [32, 40, 17, 60, 32], shape.vocab)
    pr = Pair(api, shape, 1, prompts, list(range(100, 100 + B)))
    try:
        trees = [pooled_tree(rng, n, 4, 3, shape.vocab) for n in (8, 16, 1, 32, 8)]
        trees[2] = Tree(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32))  # root-only
        a = draw_accept_lengths(rng, trees, 3.98, 1.55)
        trees = plant(trees, pr.oracle_targets(range(B)), a, shape.vocab, rng)
        batch = pr.batch(range(B), trees)
        out = api.verify(pr.model, pr.pool, batch, pr.ws, auto_commit=False)
        logits_gpu = api.debug_last_logits(pr.model, pr.ws, batch).cpu().numpy()
        g = split_outputs(out, batch)

        def run():
            ses = [OV.make_session(pr.W, p, 100 + i) for i, p in enumerate(prompts)]
            return np.concatenate([o.logits for o in OV.verify_batch(
                pr.W, [OV.Request(s_, t.parent, t.token) for s_, t in zip(ses, trees)], auto_commit=False)])
        ref_all, noise = oracle_noise_floor(run)
        bound = check_logits(logits_gpu, ref_all, noise)
        refs = OV.verify_batch(pr.W, [OV.Request(pr.sessions[r], trees[r].parent, trees[r].token) for r in range(B)],
                               auto_commit=False)
        assert all(int(x) == 0 for x in g["status"])
        check_batch(trees, refs, [o.logits for o in refs], g, bound)
        # commit through the separate entry point; committed rows == tree-scratch rows, bitwise
        L0 = [int(x) for x in pr.pool.get_len(pr.handles)]
        api.kv_commit(pr.model, pr.pool, batch, out, pr.ws)
        check_commit(api, pr.model, pr.pool, pr.ws, batch, g, pr.handles, L0)
    finally:
        pr.close()


def test_iterated_verify_commit_reproduces_greedy_decoding(api):
    """P4 on the GPU: k verify+commit steps emit the oracle's greedy continuation."""
    rng = np.random.default_rng(303)
    B = 3
    prompts = _prompts(rng, B, [32, 20, 45], TINY.vocab)
    pr = Pair(api, TINY, 1, prompts, [7, 8, 9])
    try:
        emitted_gpu = [[] for _ in range(B)]
        emitted_ref = [[] for _ in range(B)]
        exempt = 0
        for step in range(8):
            trees = [pooled_tree(rng, 8, 4, 3, TINY.vocab) for _ in range(B)]
            a = draw_accept_lengths(rng, trees, 3.98, 1.55)
            trees = plant(trees, pr.oracle_targets(range(B)), a, TINY.vocab, rng)
            batch = pr.batch(range(B), trees)
            L0 = [int(x) for x in pr.pool.get_len(pr.handles)]
            out = api.verify(pr.model, pr.pool, batch, pr.ws, auto_commit=True)
            g = split_outputs(out, batch)
            check_commit(api, pr.model, pr.pool, pr.ws, batch, g, pr.handles, L0)
            refs = OV.verify_batch(pr.W, [OV.Request(pr.sessions[r], trees[r].parent, trees[r].token)
                                          for r in range(B)])
            for r in range(B):
                kind = check_request(trees[r], refs[r], refs[r].logits, g, r)
                if kind == "exempt":
                    exempt += 1
                    pytest.skip("near-tie on a visited node; sequences diverge legitimately")
                emitted_gpu[r] += list(g["accepted_token"][r][:g["accepted_len"][r]]) + [int(g["bonus"][r])]
                emitted_ref[r] += refs[r].accepted_token + [refs[r].bonus]
            lens = pr.pool.get_len(pr.handles)
            assert list(lens) == [len(s.cache) for s in pr.sessions]
        assert emitted_gpu == emitted_ref
        # the committed caches equal the oracle's (indices exact, values within fp16 rounding)
        for r in range(B):
            s = pr.sessions[r]
            got = f16_bits_to_f64(pr.pool.read_kv(pr.handles[r], 1, 0, 0, len(s.cache)))
            assert np.abs(got - s.cache.k[1]).max() <= 0.05 * max(1.0, np.abs(s.cache.k[1]).max())
    finally:
        pr.close()


def test_verify_sampled_matches_oracle_draws(api):
    rng = np.random.default_rng(404)
    B = 4
    prompts = _prompts(rng, B, [32, 33, 34, 35], TINY.vocab)
    pr = Pair(api, TINY, 3, prompts, [1 << 40, 5, 6, 7])
    try:
        trees = [random_tree(rng, n, TINY.vocab) for n in (8, 3, 16, 0)]
        batch = pr.batch(range(B), trees, rounds=[3, 0, 9, 1 << 31])
        out = api.verify(pr.model, pr.pool, batch, pr.ws, mode=1, temperature=0.7, seed=0xDEADBEEF12345,
                         auto_commit=False)
        g = split_outputs(out, batch)
        lg = api.debug_last_logits(pr.model, pr.ws, batch).cpu().numpy()

        def run():
            return [OV.verify_one(pr.W, OV.Request(pr.sessions[r], trees[r].parent, trees[r].token, round=rnd),
                                  "sample", 0.7, 0xDEADBEEF12345) for r, rnd in enumerate([3, 0, 9, 1 << 31])]
        refs = run()
        bound = check_logits(lg, np.concatenate([o.logits for o in refs]),
                             noise_fn=lambda: oracle_noise_floor(lambda: np.concatenate([o.logits for o in run()]))[1])
        scores = [OV.target_scores(o.logits, "sample", 0.7, 0xDEADBEEF12345, rnd, pr.sessions[r].session_id)
                  for r, (o, rnd) in enumerate(zip(refs, [3, 0, 9, 1 << 31]))]
        # score error = logit error x 1/T (+ fp32 vs fp64 Gumbel transform, ~1e-6)
        check_batch(trees, refs, scores, g, bound * OV.inv_temperature(0.7) + 1e-5)
    finally:
        pr.close()


def test_errors_are_per_request_and_isolated(api):
    rng = np.random.default_rng(505)
    prompts = _prompts(rng, 4, [10, 10, 10, 10], TINY.vocab)
    pr = Pair(api, TINY, 1, prompts, [1, 2, 3, 4])
    try:
        good = pooled_tree(rng, 6, 3, 2, TINY.vocab)
        bad_parent = Tree(np.array([-1, 2, 0], np.int32), np.array([1, 2, 3], np.int32), np.zeros(3, np.float32))
        dup = Tree(np.array([-1, -1], np.int32), np.array([4, 4], np.int32), np.zeros(2, np.float32))
        bad_tok = Tree(np.array([-1], np.int32), np.array([TINY.vocab], np.int32), np.zeros(1, np.float32))
        trees = [good, bad_parent, dup, bad_tok]
        batch = pr.batch(range(4), trees)
        lens0 = pr.pool.get_len(pr.handles)
        out = api.verify(pr.model, pr.pool, batch, pr.ws, auto_commit=True)
        g = split_outputs(out, batch)
        assert list(g["status"]) == [0, 1, 4, 3]
        assert list(g["bonus"][1:]) == [-1, -1, -1] and list(g["accepted_len"][1:]) == [0, 0, 0]
        lens1 = pr.pool.get_len(pr.handles)
        assert list(lens1[1:]) == list(lens0[1:])
        o = OV.verify_one(pr.W, OV.Request(pr.sessions[0], good.parent, good.token))
        assert check_request(good, o, o.logits, g, 0) in ("exact", "exempt")
        assert lens1[0] == lens0[0] + g["accepted_len"][0] + 1
        # stale context length -> E_CONTEXT; duplicate handle -> E_HANDLE; idempotent commit
        batch2 = api.Batch.from_host([pr.handles[1], pr.handles[2], pr.handles[2]], [5, int(lens1[2]) + 1,
                                     int(lens1[2]) + 1], [1, 1, 1], [1, 2, 3], [0, 0, 0], [good, good, good])
        out2 = api.verify(pr.model, pr.pool, batch2, pr.ws, auto_commit=False)
        assert list(out2.status.cpu().numpy()) == [5, 0, 7]
        api.kv_commit(pr.model, pr.pool, batch2, out2, pr.ws)
        l_a = pr.pool.get_len([pr.handles[2]])[0]
        api.kv_commit(pr.model, pr.pool, batch2, out2, pr.ws)        # second commit: no-op
        assert pr.pool.get_len([pr.handles[2]])[0] == l_a
        assert out2.status.cpu().numpy()[1] == 5
    finally:
        pr.close()


def test_host_entry_point_equals_device_entry(api):
    rng = np.random.default_rng(606)
    prompts = _prompts(rng, 3, [20, 30, 40], TINY.vocab)
    pr = Pair(api, TINY, 1, prompts, [1, 2, 3])
    try:
        trees = [pooled_tree(rng, 8, 4, 3, TINY.vocab) for _ in range(3)]
        batch = pr.batch(range(3), trees)
        out = api.verify(pr.model, pr.pool, batch, pr.ws, auto_commit=False)
        hb = api.HostBatch.of(batch)
        ho = api.host_outputs(hb)
        api.verify_host(pr.model, pr.pool, hb, pr.ws, ho, auto_commit=False)
        for k in ("status", "accepted_len", "bonus", "row_target"):
            assert np.array_equal(getattr(out, k).cpu().numpy(), ho[k].numpy()), k
        assert api.last_launch_count() > 0
    finally:
        pr.close()


def _sampled_law_counts(api, n_draws, T, seed):
    """GPU (stop, bonus) counts for one fixed tree over many rounds, V = 16."""
    shape = TINY_V16
    W = Weights(shape, 12)
    parent = np.array([-1, -1, -1, 0, 0, 1, 3, 3], np.int32)
    token = np.array([0, 1, 2, 0, 1, 0, 0, 1], np.int32)
    B = 512
    ctx = 9
    # identical random-filled caches on every handle (same fill seed and stream id)
    cache = Cache(shape)
    for l in range(shape.n_layers):
        cache.k[l] = gen_kv_fill(99, 0, l, 0, ctx - 1, shape.n_kv, shape.head_dim)
        cache.v[l] = gen_kv_fill(99, 0, l, 1, ctx - 1, shape.n_kv, shape.head_dim)
    hf, _, _ = tree_forward(W, cache, 3, parent, token)
    logits = lm_logits(W, hf)
    law = closed_form_law(parent, token, slot_probs(logits, T))
    model = api.Model(shape, 12, max_position=1024)
    pool = api.KVPool(model, B + 4, B + 4)
    try:
        hs = []
        for _ in range(B):
            h = pool.alloc(64)
            pool.fill_random(h, ctx - 1, 99, 0)
            hs.append(h)
        ws = model.workspace(B, B * 9, 64)
        tr = Tree(parent, token, np.zeros(8, np.float32))
        counts = {}
        for k in range(n_draws // B):
            batch = api.Batch.from_host(hs, [ctx] * B, [3] * B, [42] * B, list(range(k * B, (k + 1) * B)),
                                        [tr] * B, max_context_len=64)
            out = api.verify(model, pool, batch, ws, mode=1, temperature=T, seed=seed, auto_commit=False)
            al = out.accepted_len.cpu().numpy()
            an = out.accepted_node.cpu().numpy().reshape(B, 8)
            bo = out.bonus.cpu().numpy()
            for r in range(B):
                stop = 0 if al[r] == 0 else int(an[r][al[r] - 1]) + 1
                counts[(stop, int(bo[r]))] = counts.get((stop, int(bo[r])), 0) + 1
        return counts, law
    finally:
        pool.close()
        model.close()


def test_sampled_verification_law_chi_square_on_gpu(api):
    from scipy import stats
    n = 512 * 200
    counts, law = _sampled_law_counts(api, n, 0.7, 5)
    keys = sorted(law)
    exp = np.array([law[k] * n for k in keys])
    obs = np.array([counts.get(k, 0) for k in keys], float)
    assert obs.sum() == n
    big = exp >= 5
    o = np.append(obs[big], obs[~big].sum())
    e = np.append(exp[big], exp[~big].sum())
    assert stats.chisquare(o, e * o.sum() / e.sum()).pvalue > 1e-3


def _width_slice(api, shape, seed, B, n_nodes, depth, branching, ctx_lo, ctx_hi, mode, temperature, rng_seed):
    """A bench config at full width and full vocabulary with only the layer count reduced so the
    oracle finishes: B requests x n_nodes-node pooled trees over random-filled contexts
    U[ctx_lo, ctx_hi], verified with auto_commit in the launch configuration bench.py times.
    Every slot's target, the walk, the committed KV indices and all R x V logits are compared."""
    rng = np.random.default_rng(rng_seed)
    W = Weights(shape, seed)
    cap = ctx_hi + n_nodes + 64
    model = api.Model(shape, seed, max_position=cap + 64)
    pool = api.KVPool(model, B * ((cap + 63) // 64) + 4, B)
    try:
        ctx = [int(c) for c in rng.integers(ctx_lo, ctx_hi + 1, B)]
        hs, sessions = [], []
        for r in range(B):
            h = pool.alloc(cap)
            pool.fill_random(h, ctx[r] - 1, 1234, r)
            hs.append(h)
            c = Cache(shape)
            for l in range(shape.n_layers):
                c.k[l] = gen_kv_fill(1234, r, l, 0, ctx[r] - 1, shape.n_kv, shape.head_dim)
                c.v[l] = gen_kv_fill(1234, r, l, 1, ctx[r] - 1, shape.n_kv, shape.head_dim)
            sessions.append(OV.Session(c, int(rng.integers(0, shape.vocab)), (7 << 33) + 1000 + r))
        trees = [pooled_tree(rng, n_nodes, depth, branching, shape.vocab) for _ in range(B)]
        rounds = [int(x) for x in rng.integers(0, 1 << 31, B)]
        ws = model.workspace(B, B * (n_nodes + 1), cap)
        batch = api.Batch.from_host(hs, ctx, [s.last_token for s in sessions], [s.session_id for s in sessions],
                                    rounds, trees, max_context_len=cap)
        L0 = [c - 1 for c in ctx]
        out = api.verify(model, pool, batch, ws, mode=1 if mode == "sample" else 0, temperature=temperature,
                         seed=seed, auto_commit=True)
        g = split_outputs(out, batch)
        logits_gpu = api.debug_last_logits(model, ws, batch).cpu().numpy()
        assert all(int(x) == 0 for x in g["status"])
        check_commit(api, model, pool, ws, batch, g, hs, L0)

        def run():
            return OV.verify_batch(W, [OV.Request(sessions[r], trees[r].parent, trees[r].token, round=rounds[r])
                                       for r in range(B)], mode, temperature, seed, auto_commit=False)
        refs = run()
        ref_all = np.concatenate([o.logits for o in refs])
        # the oracle's own float32-matmul deviation on the same inputs sets the max-abs bound
        bound = check_logits(logits_gpu, ref_all,
                             noise_fn=lambda: oracle_noise_floor(lambda: np.concatenate([o.logits for o in run()]))[1])
        if mode == "sample":
            scores = [OV.target_scores(o.logits, mode, temperature, seed, rounds[r], sessions[r].session_id)
                      for r, o in enumerate(refs)]
            tol = bound * OV.inv_temperature(temperature) + 1e-5
        else:
            scores, tol = [o.logits for o in refs], bound
        check_batch(trees, refs, scores, g, tol)
    finally:
        pool.close()
        model.close()


def test_full_width_two_layer_slice_matches_oracle(api):
    """cfg2 (Llama-3-8B widths: d 4096, 32/8 heads, F 14336, V 128256), 16 requests x 32-node
    trees, contexts U[768, 1280], greedy."""
    _width_slice(api, LLAMA3_8B_2L, 2, 16, 32, 7, 4, 768, 1280, "greedy", 0.0, 707)


def test_cfg3_width_two_layer_slice_matches_oracle(api):
    """cfg3 (Qwen3-14B widths: d 5120, 40/8 heads, F 17408, V 151936), one microbatch of 32
    requests x 32-node trees, contexts U[1536, 2560], greedy."""
    _width_slice(api, QWEN3_14B_2L, 3, 32, 32, 7, 4, 1536, 2560, "greedy", 0.0, 708)


def test_cfg5_width_sampled_slice_matches_oracle(api):
    """cfg5 (Qwen3-14B widths, V = 151936, SAMPLE_TREE at T = 1.0), 16 requests x 16-node trees,
    contexts U[12288, 20480] (the persistent balanced attention with in-kernel merges), Gumbel-max
    draws compared one by one with the oracle's (amb. A9)."""
    _width_slice(api, QWEN3_14B_2L, 5, 16, 16, 5, 4, 12288, 20480, "sample", 1.0, 709)


G8 = ModelShape("g8", 2, 512, 16, 2, 128, 1024, 2048, 1e-5, 500000.0)   # G = 8 (Llama-70B's group at TP 2)


@pytest.mark.parametrize("shape,sizes", [(SMALL128, (16, 32, 8, 63, 1)), (G8, (64, 20, 64, 5, 1)),
                                         (SMALL128, (16, 8, 12, 20, 1))])
def test_long_ragged_contexts_chunked_attention_matches_oracle(api, shape, sizes):
    """Long contexts (>= 64 pages) switch the tcgen05 attention to the persistent work-balanced
    grid: a 7000-token request is cut into up to 8 chunks combined by k_attn_combine, a 200-token
    one stays a single chunk written final by the attention kernel, in the same launch.  G = 8 with
    64-node trees: 5 M-tiles per request = two pair passes and a replicated single pass per item.
    Trees of <= 31 nodes (<= 128 rows per kv head): the chunks are merged inside the attention
    kernel by the last CTA of each (request, kv head) instead of the combine kernel.
    Random-filled caches (gen_kv_fill on the oracle side), every slot's target compared."""
    rng = np.random.default_rng(909)
    ctx = [4500, 200, 7000, 4100, 64]
    B = len(ctx)
    W = Weights(shape, 3)
    model = api.Model(shape, 3, max_position=8192)
    pool = api.KVPool(model, sum((c + 127) // 64 for c in ctx) + 8, B)
    try:
        hs, sessions = [], []
        for r in range(B):
            h = pool.alloc(ctx[r] + 64)
            pool.fill_random(h, ctx[r] - 1, 4321, r)
            hs.append(h)
            c = Cache(shape)
            for l in range(shape.n_layers):
                c.k[l] = gen_kv_fill(4321, r, l, 0, ctx[r] - 1, shape.n_kv, shape.head_dim)
                c.v[l] = gen_kv_fill(4321, r, l, 1, ctx[r] - 1, shape.n_kv, shape.head_dim)
            sessions.append(OV.Session(c, int(rng.integers(0, shape.vocab)), 2000 + r))
        trees = [pooled_tree(rng, n, 5, 3, shape.vocab) for n in sizes]
        ws = model.workspace(B, sum(t.n + 1 for t in trees), 7100)
        batch = api.Batch.from_host(hs, ctx, [s.last_token for s in sessions], [s.session_id for s in sessions],
                                    [0] * B, trees, max_context_len=7100)
        out = api.verify(model, pool, batch, ws, auto_commit=False)
        g = split_outputs(out, batch)
        logits_gpu = api.debug_last_logits(model, ws, batch).cpu().numpy()
        def run():
            return OV.verify_batch(W, [OV.Request(sessions[r], trees[r].parent, trees[r].token) for r in range(B)],
                                   auto_commit=False)
        refs = run()
        ref_all = np.concatenate([o.logits for o in refs])
        bound = check_logits(logits_gpu, ref_all,
                             noise_fn=lambda: oracle_noise_floor(lambda: np.concatenate([o.logits for o in run()]))[1])
        assert all(int(x) == 0 for x in g["status"])
        check_batch(trees, refs, [o.logits for o in refs], g, bound)
    finally:
        pool.close()
        model.close()


def test_verify_is_bitwise_deterministic(api):
    """Two verifies of the same batch give bit-identical logits, targets and scores: every
    reduction has a fixed order (K-split partials summed in split order by the consumer, split-KV
    chunks merged in chunk order — also by whichever CTA of the balanced attention finishes last)."""
    shape = SMALL128
    rng = np.random.default_rng(4242)
    ctx = [5000, 300, 6100, 64]
    B = len(ctx)
    model = api.Model(shape, 5, max_position=8192)
    pool = api.KVPool(model, sum((c + 127) // 64 for c in ctx) + 8, B)
    try:
        hs = []
        for r in range(B):
            h = pool.alloc(ctx[r] + 64)
            pool.fill_random(h, ctx[r] - 1, 99, r)
            hs.append(h)
        trees = [pooled_tree(rng, n, 5, 3, shape.vocab) for n in (20, 8, 31, 1)]   # <= 128 rows/kv head
        ws = model.workspace(B, sum(t.n + 1 for t in trees), 6200)
        batch = api.Batch.from_host(hs, ctx, [3] * B, [500 + r for r in range(B)], [0] * B, trees,
                                    max_context_len=6200)
        runs = []
        for _ in range(2):
            out = api.verify(model, pool, batch, ws, mode=api.L.SAMPLE_TREE, temperature=1.0, seed=3,
                             auto_commit=False)
            lg = api.debug_last_logits(model, ws, batch).cpu().numpy()
            runs.append((lg.view(np.uint32).copy(), out.row_target.cpu().numpy().copy(),
                         out.row_score.cpu().numpy().view(np.uint32).copy()))
        for a, b in zip(runs[0], runs[1]):
            assert np.array_equal(a, b)
    finally:
        pool.close()
        model.close()
