"""Oracle for SURVEY §8(f) NEXT-F2: dense-q speculative sampling of a *sampled* draft chain.

PAPER.md App. B: "we implemented the speculative decoding technique from
[Leviathan et al. 2023], which uses a linear candidate sequence"; the edge samples each draft token
from its draft distribution q and ships q with it (the dense-q wire variant).
SPEC.md S:184 fixes the single-node arithmetic (accept x with probability min(1, p(x)/q(x)); on
rejection the bonus comes from norm(max(0, p - q))).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): plain numpy float64, shares nothing with
paper_2505_17052_b200/csrc.

Algorithm (per request; slots s = 0..N, slot 0 = root, node i = slot i+1 is the child of slot i):
  cur = slot 0
  for i in 0..N-1:                                  node i's token x was drawn from q_i = q[slot i]
      p = softmax(l[slot i] / T)
      accept node i iff u(slot i) < p(x) / q_i(x)   (Leviathan: probability min(1, p/q))
      else: bonus ~ norm(max(0, p - q_i)), stop
  if every node was accepted: bonus ~ p at the last slot
Random numbers (readings, DESIGN.md §4 R-pq):
  u(slot) = ((w >> 8) | 1) * 2^-24 with w = Philox word 0 of counter (slot, 'ACPT', lo32(session),
            hi32(session)), key (lo32(seed) ^ round, hi32(seed)) — exact, in (0, 1);
  bonus draws are Gumbel-max with the SAMPLE_TREE noise g(seed, round, session, slot, v)
  (oracle/verify.py:gumbel): argmax_v (log r_v + g_v) over r_v > 0 samples norm(r).
"""
from __future__ import annotations

import itertools

import numpy as np

from . import philox
from .verify import (Outcome, OK, E_TREE, gumbel, inv_temperature, validate, walk,  # noqa: F401
                     commit)
from .model import tree_forward, lm_logits

ACCEPT_TAG = 0x41435054   # 'ACPT'


def accept_uniform(seed, round_, session, slot):
    lo, hi = philox.split_seed(seed)
    s_lo, s_hi = philox.split_seed(session)
    r = philox.philox4x32_10(np.uint64(slot), ACCEPT_TAG, s_lo, s_hi, lo ^ (int(round_) & 0xFFFFFFFF), hi)
    w = int(np.asarray(r[0]).reshape(-1)[0])
    return float(((w >> 8) | 1) * 2.0 ** -24)


def softmax_t(logits_row, invT):
    z = np.asarray(logits_row, np.float64) * invT
    z = z - z.max()
    e = np.exp(z)
    return e / e.sum()


def chain_walk(p_rows, q_rows, tokens, uniforms, noise):
    """The decision logic on explicit distributions: p_rows [N+1, V], q_rows [N, V] (q_rows[i] is the
    distribution node i was drawn from), tokens [N], uniforms [N], noise(slot) -> [V] Gumbel.
    Returns (accepted node indices, bonus, stop slot, ratios)."""
    n = len(tokens)
    acc, ratios = [], []
    for i in range(n):
        x = int(tokens[i])
        p, q = p_rows[i], q_rows[i]
        ratio = p[x] / q[x] if q[x] > 0 else np.inf
        ratios.append(ratio)
        if uniforms[i] < ratio:
            acc.append(i)
            continue
        r = np.maximum(0.0, p - q)
        score = np.where(r > 0, np.log(np.where(r > 0, r, 1.0)) + noise(i), -np.inf)
        return acc, int(np.argmax(score)), i, ratios
    return acc, int(np.argmax(np.log(np.maximum(p_rows[n], 1e-300)) + noise(n))), n, ratios


def exact_chain_law(p_fn, q_fn, depth, vocab, horizon=None):
    """Exact distribution of the first `horizon` (default depth+1) emitted tokens of one verify round
    of a chain of `depth` tokens drawn from q, completed autoregressively from p when the round
    emits fewer tokens.  p_fn(prefix) / q_fn(prefix) -> probability vectors.  Returns a dict
    sequence -> probability.  Used to pin chain_walk's rule against the target AR law."""
    H = horizon or depth + 1
    out = {}

    def complete(prefix, prob):
        if len(prefix) >= H:
            key = tuple(prefix[:H])
            out[key] = out.get(key, 0.0) + prob
            return
        p = p_fn(tuple(prefix))
        for v in range(vocab):
            if p[v] > 0:
                complete(prefix + [v], prob * p[v])

    def step(prefix, k, prob):
        # position k of the round: draft token x ~ q(.|prefix), accepted w.p. min(1, p/q)
        if k == depth:   # all accepted: bonus ~ p
            complete(prefix, prob)
            return
        p, q = p_fn(tuple(prefix)), q_fn(tuple(prefix))
        resid = np.maximum(0.0, p - q)
        z = resid.sum()
        for x in range(vocab):
            if q[x] <= 0:
                continue
            a = min(1.0, p[x] / q[x])
            if a > 0:
                step(prefix + [x], k + 1, prob * q[x] * a)
            if a < 1 and z > 0:
                for v in range(vocab):
                    if resid[v] > 0:
                        complete(prefix + [v], prob * q[x] * (1 - a) * resid[v] / z)

    step([], 0, 1.0)
    return out


def ar_law(p_fn, vocab, horizon):
    out = {}
    for seq in itertools.product(range(vocab), repeat=horizon):
        pr = 1.0
        for i in range(horizon):
            pr *= p_fn(tuple(seq[:i]))[seq[i]]
        if pr > 0:
            out[seq] = pr
    return out


def is_chain(parent):
    return all(int(p) == i - 1 for i, p in enumerate(parent))


E_UNSUPPORTED = 8   # SPECEDGE_REQ_E_UNSUPPORTED: dense-q mode needs a chain


def verify_pq(W, reqs, draft_q, temperature, seed, auto_commit=True):
    """Dense-q verification of a batch of sampled chains.  draft_q[r] is [N_r, V] (row i = the
    distribution node i was drawn from).  Returns oracle/verify.py Outcome objects (row_target =
    the bonus draw of each slot's would-be stop, for inspection: slot s < N -> residual draw,
    slot N -> p draw) plus .ratios / .stop attributes."""
    s = W.shape
    invT = inv_temperature(temperature)
    outs = []
    for req, q in zip(reqs, draft_q):
        ses = req.session
        parent = [int(x) for x in req.parent]
        token = [int(x) for x in req.token]
        st = validate(parent, token, ses.last_token, s.vocab, ses.context_len, len(ses.cache))
        if st == OK and not is_chain(parent):
            st = E_UNSUPPORTED
        if st != OK:
            outs.append(Outcome(status=st))
            continue
        hf, tk, tv = tree_forward(W, ses.cache, ses.last_token, parent, token)
        logits = lm_logits(W, hf)
        p_rows = np.stack([softmax_t(l, invT) for l in logits])
        n = len(token)
        u = [accept_uniform(seed, ses.round, ses.session_id, i) for i in range(n)]

        def noise(slot):
            return gumbel(seed, ses.round, ses.session_id, slot, s.vocab)
        acc, bonus, stop, ratios = chain_walk(p_rows, np.asarray(q, np.float64), token, u, noise)
        o = Outcome(OK, [token[i] for i in acc], acc, bonus, None, None, logits, tk, tv)
        o.ratios, o.stop, o.uniforms, o.p_rows = ratios, stop, u, p_rows
        outs.append(o)
    if auto_commit:
        for r, o in zip(reqs, outs):
            if o.status == OK:
                commit(r.session, o)
    return outs
