"""Pins of the oracle's verification path against plain definitions:
brute-force causal decoding, textbook causal prefill, greedy autoregressive decoding, the
closed-form law of lossless sampling, an independent rejection-sampling formulation."""
import json
import os

import numpy as np
import pytest
from scipy import stats

from oracle import verify as V
from oracle.law import closed_form_law, rejection_law, slot_probs
from oracle.model import Cache, Weights, decode, prefill_dense, tree_forward, lm_logits, tree_depth
from synth.configs import TINY, TINY_V16, TINY_MHA
from synth.trees import random_tree, chain_tree, pooled_tree, Tree
from synth.plant import plant

HERE = os.path.dirname(__file__)


def _prompt(rng, n, vocab):
    return [int(t) for t in rng.integers(0, vocab, n)]


def _greedy_targets(W, sessions):
    def targets(trees):
        out = []
        for ses, t in zip(sessions, trees):
            o = V.verify_one(W, V.Request(ses, t.parent, t.token), keep_logits=False)
            out.append(o.row_target)
        return out
    return targets


# ---------------------------------------------------------------- worked example (golden) ----
def test_worked_example_fixture():
    g = json.load(open(os.path.join(HERE, "golden", "worked_example.json")))
    parent, token = g["parent"], g["token"]
    assert list(tree_depth(parent)) == g["depth"]
    L = g["cache_len"]
    assert [L] + [L + d for d in tree_depth(parent)] == g["pos_slots"]
    assert V.ancestor_masks(parent) == g["anc"]
    acc_t, acc_n, bonus = V.walk(parent, token, g["y"])
    assert (len(acc_t), acc_t, acc_n, bonus) == (g["accepted_len"], g["accepted_token"],
                                                 g["accepted_node"], g["bonus"])
    assert [0] + [n + 1 for n in acc_n] == g["commit_src_slots"]
    assert [L + j for j in range(len(acc_n) + 1)] == g["commit_dst_pos"]
    assert L + len(acc_n) + 1 == g["new_cache_len"]
    y2 = list(g["y"])
    y2[0] = g["variant_root_mismatch"]["y0"]
    a2 = V.walk(parent, token, y2)
    assert (len(a2[0]), a2[2]) == (g["variant_root_mismatch"]["accepted_len"], g["variant_root_mismatch"]["bonus"])
    a3 = V.walk([], [], g["variant_empty_tree"]["y"])
    assert (len(a3[0]), a3[2]) == (0, g["variant_empty_tree"]["bonus"])


# ------------------------------------------------------------------------ P1: tree == paths ----
@pytest.mark.parametrize("shape,n", [(TINY, 0), (TINY, 1), (TINY, 9), (TINY, 64), (TINY_MHA, 12)])
def test_tree_forward_equals_per_path_causal_decoding(shape, n):
    rng = np.random.default_rng(10 + n)
    W = Weights(shape, 7)
    prompt = _prompt(rng, 12, shape.vocab)
    ses = V.make_session(W, prompt, 1)
    tree = random_tree(rng, n, shape.vocab)
    hf, tk, tv = tree_forward(W, ses.cache, ses.last_token, tree.parent, tree.token)
    for slot in range(n + 1):
        path = []
        cur = slot - 1
        while cur >= 0:
            path.append(int(tree.token[cur]))
            cur = int(tree.parent[cur])
        seq = [ses.last_token] + path[::-1]
        c = ses.cache.copy()
        ref = decode(W, c, seq)
        assert np.allclose(hf[slot], ref[-1], rtol=0, atol=1e-9), slot
        for l in range(shape.n_layers):
            assert np.allclose(tk[l][slot], c.k[l][-1], atol=1e-9)
            assert np.allclose(tv[l][slot], c.v[l][-1], atol=1e-9)


# ---------------------------------------------------------------- P2: chain == causal prefill ----
def test_chain_tree_equals_dense_causal_prefill():
    rng = np.random.default_rng(20)
    W = Weights(TINY, 3)
    seq = _prompt(rng, 30, TINY.vocab)
    hf_ref, cache_ref = prefill_dense(W, seq)
    ses = V.make_session(W, seq[:10], 2)          # caches seq[:9], root = seq[9]
    hf, tk, tv = tree_forward(W, ses.cache, ses.last_token, chain_tree(seq[10:]).parent, seq[10:])
    assert np.allclose(hf, hf_ref[9:], atol=1e-9)
    for l in range(TINY.n_layers):
        assert np.allclose(tk[l], cache_ref.k[l][9:], atol=1e-9)
    # and the one-token-at-a-time decoder agrees with the dense prefill
    c = Cache(TINY)
    hf_dec = decode(W, c, seq)
    assert np.allclose(hf_dec, hf_ref, atol=1e-9)


# --------------------------------------------------------------------- P3: root-only verify ----
def test_root_only_is_one_autoregressive_step():
    rng = np.random.default_rng(30)
    W = Weights(TINY, 4)
    prompt = _prompt(rng, 16, TINY.vocab)
    ses = V.make_session(W, prompt, 3)
    out = V.verify_one(W, V.Request(ses, np.zeros(0, np.int32), np.zeros(0, np.int32)))
    c = ses.cache.copy()
    ref = lm_logits(W, decode(W, c, [ses.last_token]))
    assert out.accepted_len == 0 and out.bonus == int(np.argmax(ref[-1]))


# -------------------------------------------------------------- P4: greedy losslessness ----
@pytest.mark.parametrize("kind", ["random", "planted", "pooled"])
def test_greedy_verify_reproduces_greedy_decoding(kind):
    rng = np.random.default_rng(40)
    W = Weights(TINY, 5)
    prompt = _prompt(rng, 20, TINY.vocab)
    ses = V.make_session(W, prompt, 4)
    # reference: textbook greedy autoregressive continuation
    c = ses.cache.copy()
    tok = ses.last_token
    ref = []
    for _ in range(40):
        h = decode(W, c, [tok])
        tok = int(np.argmax(lm_logits(W, h)[-1]))
        ref.append(tok)
    emitted = []
    steps = 0
    while len(emitted) < 30:
        if kind == "random":
            tree = random_tree(rng, 12, TINY.vocab)
        else:
            tree = pooled_tree(rng, 12, 4, 3, TINY.vocab)
            if kind == "planted":
                a = int(rng.integers(0, 4))
                tree = plant([tree], _greedy_targets(W, [ses]), [a], TINY.vocab, rng)[0]
        out = V.verify_batch(W, [V.Request(ses, tree.parent, tree.token)])[0]
        assert out.status == V.OK
        emitted += out.accepted_token + [out.bonus]
        steps += 1
    assert emitted[:30] == ref[:30]
    if kind == "planted":
        assert steps < 30          # planting produced multi-token steps


# ------------------------------------------------------- P5 / P6: full accept, no match ----
def test_draft_equal_to_greedy_continuation_is_fully_accepted():
    rng = np.random.default_rng(50)
    W = Weights(TINY, 6)
    ses = V.make_session(W, _prompt(rng, 10, TINY.vocab), 5)
    c = ses.cache.copy()
    tok, cont = ses.last_token, []
    for _ in range(7):
        tok = int(np.argmax(lm_logits(W, decode(W, c, [tok]))[-1]))
        cont.append(tok)
    out = V.verify_one(W, V.Request(ses, chain_tree(cont[:6]).parent, cont[:6]))
    assert out.accepted_token == cont[:6] and out.bonus == cont[6]
    # P6: no child of the root matches -> a = 0, bonus = y[root]
    bad = [(cont[0] + 1) % TINY.vocab, (cont[0] + 2) % TINY.vocab]
    out2 = V.verify_one(W, V.Request(ses, np.array([-1, -1]), np.array(bad)))
    assert out2.accepted_len == 0 and out2.bonus == cont[0]


# ------------------------------------------------------------------- P10: commit == prefill ----
def test_commit_equals_fresh_prefill():
    rng = np.random.default_rng(60)
    W = Weights(TINY, 8)
    prompt = _prompt(rng, 14, TINY.vocab)
    ses = V.make_session(W, prompt, 6)
    tree = plant([pooled_tree(rng, 16, 5, 3, TINY.vocab)], _greedy_targets(W, [ses]), [3],
                 TINY.vocab, rng)[0]
    L0 = len(ses.cache)
    out = V.verify_batch(W, [V.Request(ses, tree.parent, tree.token)])[0]
    assert out.accepted_len == 3
    assert len(ses.cache) == L0 + out.accepted_len + 1
    _, cache_ref = prefill_dense(W, prompt + out.accepted_token)
    for l in range(TINY.n_layers):
        assert np.allclose(ses.cache.k[l], cache_ref.k[l], atol=1e-9)
        assert np.allclose(ses.cache.v[l], cache_ref.v[l], atol=1e-9)
    assert ses.last_token == out.bonus and ses.context_len == len(prompt) + 4


# ------------------------------------------------------------ P11 / P12: batch/solo, replay ----
def test_batch_equals_solo_and_replay_is_deterministic():
    rng = np.random.default_rng(70)
    W = Weights(TINY, 9)
    prompts = [_prompt(rng, int(n), TINY.vocab) for n in rng.integers(3, 25, 4)]
    trees = [random_tree(rng, int(n), TINY.vocab) for n in (0, 5, 17, 64)]
    mk = lambda: [V.make_session(W, p, 100 + i) for i, p in enumerate(prompts)]
    for mode, T in (("greedy", 0.0), ("sample", 0.7)):
        ses_b = mk()
        batch = V.verify_batch(W, [V.Request(s, t.parent, t.token) for s, t in zip(ses_b, trees)],
                               mode, T, seed=11, auto_commit=False)
        for i, (p, t) in enumerate(zip(prompts, trees)):
            solo = V.verify_one(W, V.Request(V.make_session(W, p, 100 + i), t.parent, t.token),
                                mode, T, seed=11)
            assert (solo.accepted_token, solo.accepted_node, solo.bonus) == \
                   (batch[i].accepted_token, batch[i].accepted_node, batch[i].bonus)
            assert np.array_equal(solo.row_target, batch[i].row_target)
    # changing round changes the Gumbel draws (P12)
    g1 = V.gumbel(11, 0, 100, 3, 256)
    assert np.array_equal(g1, V.gumbel(11, 0, 100, 3, 256))
    assert not np.array_equal(g1, V.gumbel(11, 1, 100, 3, 256))
    assert not np.array_equal(g1, V.gumbel(11, 0, 101, 3, 256))
    assert not np.array_equal(g1, V.gumbel(11, 0, 100, 4, 256))


# --------------------------------------------------------------------- validation (A5, A18) ----
def test_per_request_validation_codes_and_isolation():
    rng = np.random.default_rng(80)
    W = Weights(TINY, 10)
    good = V.make_session(W, _prompt(rng, 8, TINY.vocab), 1)
    mk = lambda: V.make_session(W, _prompt(np.random.default_rng(81), 8, TINY.vocab), 2)
    cases = [
        (dict(parent=[-1, 1], token=[1, 2]), V.E_TREE),
        (dict(parent=[-1, 5], token=[1, 2]), V.E_TREE),
        (dict(parent=[-1] * 65, token=list(range(65))), V.E_TREE_SIZE),
        (dict(parent=[-1, 0], token=[1, 256]), V.E_TOKEN),
        (dict(parent=[-1, -1], token=[3, 3]), V.E_DUP_SIBLING),
        (dict(parent=[-1, 0, 0], token=[3, 4, 4]), V.E_DUP_SIBLING),
        (dict(parent=[-1], token=[3], context_len=3), V.E_CONTEXT),
    ]
    for kw, code in cases:
        ses = mk()
        L = len(ses.cache)
        req = V.Request(ses, np.array(kw["parent"]), np.array(kw["token"]),
                        context_len=kw.get("context_len", -1))
        ok_req = V.Request(good, np.array([-1]), np.array([5]))
        outs = V.verify_batch(W, [req, ok_req])
        assert outs[0].status == code and outs[0].accepted_len == 0 and outs[0].bonus == -1
        assert len(ses.cache) == L                      # no commit for the errored request
        assert outs[1].status == V.OK
    # sibling tokens may repeat across different parents
    assert V.validate([-1, 0, 1], [3, 3, 3], 0, 256, 5, 4) == V.OK


# ----------------------------------------------------------- P8: Gumbel marginals = softmax ----
@pytest.mark.parametrize("T", [0.5, 0.7, 1.0, 2.0])
def test_gumbel_max_marginal_equals_softmax(T):
    rng = np.random.default_rng(90)
    V_ = 16
    logits = rng.standard_normal((1, V_)) * 2.0
    n = 40000
    counts = np.zeros(V_)
    for r in range(n):
        counts[int(np.argmax(V.target_scores(logits, "sample", T, 5, r, 77)[0]))] += 1
    p = slot_probs(logits, T)[0]
    keep = p * n >= 5
    obs = np.append(counts[keep], counts[~keep].sum())
    exp = np.append(p[keep] * n, p[~keep].sum() * n)
    if exp[-1] == 0:
        obs, exp = obs[:-1], exp[:-1]
    assert stats.chisquare(obs, exp).pvalue > 1e-3


# --------------------------------------------- P9: rejection form (O8) == closed form (O7) ----
def test_rejection_form_law_equals_closed_form_exactly():
    rng = np.random.default_rng(100)
    for trial in range(20):
        n = int(rng.integers(0, 10))
        tree = random_tree(rng, n, 6)
        probs = rng.dirichlet(np.ones(6) * 0.7, n + 1)
        a = closed_form_law(tree.parent, tree.token, probs)
        for key in (None, lambda c: (-tree.logprob[c], tree.token[c]), lambda c: -c):
            b = rejection_law(tree.parent, tree.token, probs, key)
            ks = set(a) | set(b)
            tv = 0.5 * sum(abs(a.get(k, 0.0) - b.get(k, 0.0)) for k in ks)
            assert tv < 1e-12
        assert abs(sum(a.values()) - 1.0) < 1e-12


# ------------------------------------------- P7: chi-square of the sampled law (V = 16) ----
def _sampled_outcomes(logits, parent, token, T, n_rounds, seed, session, sampler="gumbel"):
    S, V_ = logits.shape
    rounds = np.arange(n_rounds)
    Teff = T if sampler == "gumbel" else 1.0     # "wrong": ignores the temperature (power check)
    invT = V.inv_temperature(Teff)
    ys = np.stack([np.argmax(logits[s] * invT + V.gumbel(seed, rounds, session, s, V_), axis=-1)
                   for s in range(S)], axis=1)
    # the vectorised draw equals the per-round reference formulation
    for r in (0, 1, n_rounds - 1):
        assert np.array_equal(ys[r], np.argmax(V.target_scores(logits, "sample", Teff, seed, r, session), -1))
    counts = {}
    for r in range(n_rounds):
        acc_t, acc_n, bonus = V.walk(parent, token, ys[r])
        stop = 0 if not acc_n else acc_n[-1] + 1
        counts[(stop, bonus)] = counts.get((stop, bonus), 0) + 1
    return counts


def _chi2(counts, law, n):
    keys = sorted(law)
    exp = np.array([law[k] * n for k in keys])
    obs = np.array([counts.get(k, 0) for k in keys], float)
    assert sum(counts.values()) == obs.sum()          # no outcome outside the law's support
    big = exp >= 5
    o = np.append(obs[big], obs[~big].sum())
    e = np.append(exp[big], exp[~big].sum())
    return stats.chisquare(o, e * o.sum() / e.sum()).pvalue


@pytest.mark.slow
def test_stochastic_verification_law_chi_square():
    rng = np.random.default_rng(110)
    W = Weights(TINY_V16, 12)
    ses = V.make_session(W, _prompt(rng, 9, 16), 9)
    parent = np.array([-1, -1, -1, 0, 0, 1, 3, 3])
    tree = Tree(parent, np.zeros(8, np.int32), np.zeros(8, np.float32))
    # distinct sibling tokens, chosen among each slot's likely tokens so deep paths get mass
    out0 = V.verify_one(W, V.Request(ses, parent, np.array([0, 1, 2, 0, 1, 0, 0, 1])))
    T = 0.7                                                   # P:353 temperature
    probs0 = slot_probs(out0.logits, T)
    tok = np.zeros(8, np.int32)
    for node in range(8):
        ps = 0 if parent[node] < 0 else parent[node] + 1
        used = {int(tok[c]) for c in range(node) if parent[c] == parent[node]}
        order = [int(v) for v in np.argsort(-probs0[ps]) if int(v) not in used]
        tok[node] = order[0]
    hf, _, _ = tree_forward(W, ses.cache, ses.last_token, parent, tok)
    logits = lm_logits(W, hf)
    law = closed_form_law(parent, tok, slot_probs(logits, T))
    n = 200000
    counts = _sampled_outcomes(logits, parent, tok, T, n, 5, 9)
    assert _chi2(counts, law, n) > 1e-3
    # power: the same test rejects a sampler with the wrong temperature
    bad = _sampled_outcomes(logits, parent, tok, T, 20000, 5, 9, sampler="wrong")
    assert _chi2(bad, law, 20000) < 1e-6
