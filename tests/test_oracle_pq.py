"""Pins of the NEXT-F2 oracle (oracle/pq.py, dense-q speculative sampling of a sampled chain,
PAPER.md App. B) against what the mathematics fixes:
  * S:184's worked example (acceptance 1/2, residual [1,0,0,0]);
  * exact enumeration: one verify round + autoregressive completion has exactly the target's
    autoregressive law (Leviathan et al.'s theorem), TV < 1e-12, for random tables with V = 4;
  * the sampled implementation (Philox uniforms + Gumbel bonus draws) matches that exact law
    (chi-square over 6e4 draws) and a wrong rule (no residual, bonus ~ p) is rejected;
  * draft == target accepts everything; the uniform is exact and in (0, 1)."""
import numpy as np
from scipy import stats

from oracle import pq
from oracle.verify import gumbel


def _tables(rng, vocab, alpha=0.7, zeros=False):
    cache_p, cache_q = {}, {}

    def mk(cache, prefix):
        if prefix not in cache:
            d = rng.dirichlet(np.full(vocab, alpha))
            if zeros and rng.random() < 0.3:
                d[rng.integers(vocab)] = 0.0
                d /= d.sum()
            cache[prefix] = d
        return cache[prefix]
    return (lambda pre: mk(cache_p, pre)), (lambda pre: mk(cache_q, pre))


def test_spec_worked_example():
    p = np.array([0.5, 0.25, 0.125, 0.125])
    q = np.full(4, 0.25)
    # accepted iff u < p(3)/q(3) = 1/2; on rejection the residual is [1,0,0,0] -> bonus 0
    acc, bonus, stop, ratios = pq.chain_walk(np.stack([p, p]), q[None], [3], [0.49], lambda s: np.zeros(4))
    assert acc == [0] and ratios == [0.5]
    acc, bonus, stop, _ = pq.chain_walk(np.stack([p, p]), q[None], [3], [0.51], lambda s: np.zeros(4))
    assert acc == [] and bonus == 0 and stop == 0
    # for ANY Gumbel noise the residual draw is 0 (the only positive residual entry)
    rng = np.random.default_rng(1)
    for _ in range(50):
        _, bonus, _, _ = pq.chain_walk(np.stack([p, p]), q[None], [3], [0.9], lambda s: rng.gumbel(size=4))
        assert bonus == 0


def test_exact_law_equals_target_autoregressive_law():
    rng = np.random.default_rng(7)
    for trial in range(40):
        vocab = 4 if trial % 2 else 3
        depth = 1 + trial % 3
        p_fn, q_fn = _tables(rng, vocab, alpha=0.5 + trial % 3, zeros=trial % 4 == 0)
        law = pq.exact_chain_law(p_fn, q_fn, depth, vocab)
        ar = pq.ar_law(p_fn, vocab, depth + 1)
        keys = set(law) | set(ar)
        tv = 0.5 * sum(abs(law.get(k, 0.0) - ar.get(k, 0.0)) for k in keys)
        assert tv < 1e-12, (trial, tv)
        assert abs(sum(law.values()) - 1.0) < 1e-12


def test_draft_equal_target_accepts_everything():
    rng = np.random.default_rng(3)
    p = rng.dirichlet(np.ones(16), size=5)
    toks = [int(rng.choice(16, p=p[i])) for i in range(4)]
    acc, bonus, stop, ratios = pq.chain_walk(p, p[:4], toks, [1 - 2 ** -24] * 4, lambda s: rng.gumbel(size=16))
    assert acc == [0, 1, 2, 3] and stop == 4 and all(abs(r - 1) < 1e-15 for r in ratios)


def test_accept_uniform_exact_and_in_open_interval():
    vals = [pq.accept_uniform(s, r, ses, sl) for s in (0, 5) for r in (0, 1, 2**32 - 1) for ses in (0, 2**63)
            for sl in (0, 63)]
    for v in vals:
        assert 0.0 < v < 1.0
        assert v * 2 ** 24 == int(v * 2 ** 24)     # a multiple of 2^-24: exact
    assert len(set(vals)) == len(vals)


def test_sampled_rule_matches_exact_law_chi_square():
    """The oracle's sampled implementation (Philox uniforms, Gumbel-max bonus) on a V = 4 depth-2
    chain: the first 3 emitted tokens (round + autoregressive completion from p) follow the exact
    law; a rule that drops the residual (bonus ~ p after a rejection) is rejected."""
    rng = np.random.default_rng(11)
    V, depth = 4, 2
    p_fn, q_fn = _tables(rng, V, alpha=0.8)
    law = pq.exact_chain_law(p_fn, q_fn, depth, V)
    n_draws = 60_000
    sampler = np.random.default_rng(12)
    counts, bad_counts = {}, {}
    seed, session = 9, 1234
    for rnd in range(n_draws):
        # drafts drawn from q (the edge), then the verifier's own Philox / Gumbel draws
        toks, pre = [], ()
        for _ in range(depth):
            x = int(sampler.choice(V, p=q_fn(pre)))
            toks.append(x)
            pre = pre + (x,)
        p_rows = np.stack([p_fn(tuple(toks[:i])) for i in range(depth + 1)])
        q_rows = np.stack([q_fn(tuple(toks[:i])) for i in range(depth)])
        u = [pq.accept_uniform(seed, rnd, session, i) for i in range(depth)]
        noise = lambda s: gumbel(seed, rnd, session, s, V)  # noqa: E731
        acc, bonus, stop, _ = pq.chain_walk(p_rows, q_rows, toks, u, noise)
        emitted = [toks[i] for i in acc] + [bonus]
        while len(emitted) < depth + 1:
            emitted.append(int(sampler.choice(V, p=p_fn(tuple(emitted)))))
        counts[tuple(emitted[:depth + 1])] = counts.get(tuple(emitted[:depth + 1]), 0) + 1
        # wrong rule: after a rejection draw the bonus from p instead of the residual
        if stop < depth:
            wrong = [toks[i] for i in acc] + [int(np.argmax(np.log(p_rows[stop]) + noise(stop)))]
        else:
            wrong = emitted[:len(acc) + 1]
        while len(wrong) < depth + 1:
            wrong.append(int(sampler.choice(V, p=p_fn(tuple(wrong)))))
        bad_counts[tuple(wrong[:depth + 1])] = bad_counts.get(tuple(wrong[:depth + 1]), 0) + 1

    def chi2(cnt):
        keys = sorted(law)
        exp = np.array([law[k] * n_draws for k in keys])
        obs = np.array([cnt.get(k, 0) for k in keys], float)
        big = exp >= 5
        o = np.append(obs[big], obs[~big].sum())
        e = np.append(exp[big], exp[~big].sum())
        if e[-1] == 0:
            o, e = o[:-1], e[:-1]
        return stats.chisquare(o, e).pvalue
    assert chi2(counts) > 1e-3
    assert chi2(bad_counts) < 1e-6
