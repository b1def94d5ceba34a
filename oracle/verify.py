"""Verification of draft trees: target token per slot, accept walk, bonus, KV commit.

Follows P:171 (§4.1: the server "verifies them in a single forward pass ... returns both the
verified tokens and one additional token", preserving "the exact output distribution of the
server model"), P:315-316 (§4.3 heterogeneous batches, per-sequence masks), and the readings
SURVEY §8(c) O3-O5, amb. A5-A10, A17-A22:

  O3  GREEDY: y[s] = argmax_v l[s, v], ties -> lowest v.
      SAMPLE: y[s] = argmax_v (l[s, v] * invT + g(seed, round, session, s, v)) (Gumbel-max,
              amb. A7-A9), invT = f32(1/T); T < 1e-6 -> GREEDY.
  O4  walk: cur = root; while some child c of cur has token(c) == y[cur]: accept c, cur = c;
      bonus = y[cur] (P:171 'one additional token'; amb. A10: always emitted).
  O5  commit: cache gets K/V of the root and of every accepted node, in path order; the next
      root is the bonus (amb. A19).

Per-request validation (amb. A5, A18): status codes below; an errored request gets
accepted_len 0, bonus -1, no commit, and does not affect the others.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import philox
from .model import Cache, Weights, tree_forward, lm_logits, tree_depth

OK, E_TREE, E_TREE_SIZE, E_TOKEN, E_DUP_SIBLING, E_CONTEXT = 0, 1, 2, 3, 4, 5
MAX_NODES = 64


def validate(parent, token, root_token, vocab, context_len, cache_len):
    """amb. A5: parent[i] in {-1} U [0, i); N <= 64; tokens in [0, V); sibling tokens distinct;
    context_len == cached + 1 (S:181 'context-length mismatch -> protocol error').  The first
    failing check, in this order, decides the code."""
    n = len(parent)
    if n > MAX_NODES:
        return E_TREE_SIZE
    for i, p in enumerate(parent):
        if not (p == -1 or 0 <= p < i):
            return E_TREE
    if not (0 <= root_token < vocab) or any(not (0 <= t < vocab) for t in token):
        return E_TOKEN
    seen = set()
    for p, t in zip(parent, token):
        if (int(p), int(t)) in seen:
            return E_DUP_SIBLING
        seen.add((int(p), int(t)))
    if context_len != cache_len + 1:
        return E_CONTEXT
    return OK


def ancestor_masks(parent):
    """Ancestor-or-self bitmask over node bits (root implicit): anc[i] = anc[parent[i]] | 1<<i."""
    anc = []
    for i, p in enumerate(parent):
        anc.append((0 if p < 0 else anc[p]) | (1 << i))
    return anc


def gumbel(seed, round_, session, slot, vocab):
    """amb. A9: key (lo32(seed) ^ round, hi32(seed)); counter (v>>2, slot, lo32(session),
    hi32(session)); word v&3; u = ((x>>8)|1) * 2^-24 in (0,1) exactly; g = -log(-log u)."""
    lo, hi = philox.split_seed(seed)
    s_lo, s_hi = philox.split_seed(session)
    if np.ndim(round_) == 0:
        w = philox.words_range(0, vocab, slot, s_lo, s_hi, lo ^ (int(round_) & 0xFFFFFFFF), hi)
    else:   # many rounds at once -> [n_rounds, vocab]
        k0 = (np.asarray(round_, np.uint64) & np.uint64(0xFFFFFFFF)) ^ np.uint64(lo)
        ctr = np.arange((vocab + 3) // 4, dtype=np.uint64)[None, :]
        r = philox.philox4x32_10(ctr, slot, s_lo, s_hi, k0[:, None], hi)
        w = np.stack(r, axis=-1).reshape(k0.shape[0], -1)[:, :vocab]
    u = ((w >> np.uint64(8)) | np.uint64(1)).astype(np.float64) * 2.0 ** -24
    return -np.log(-np.log(u))


def inv_temperature(T):
    return float(np.float32(1.0 / float(T)))


def target_scores(logits, mode, temperature, seed, round_, session):
    """Per-slot score rows whose argmax is y (O3).  logits [S, V]."""
    if mode == "greedy" or temperature < 1e-6:
        return np.asarray(logits, np.float64)
    invT = inv_temperature(temperature)
    S, V = logits.shape
    g = np.stack([gumbel(seed, round_, session, s, V) for s in range(S)])
    return logits * invT + g


def argmax_lowest(scores):
    """argmax along the last axis, ties -> lowest index (np.argmax returns the first maximum)."""
    return np.argmax(scores, axis=-1)


def walk(parent, token, y):
    """O4.  y[slot] for slot 0 = root, i+1 = node i.  Returns (acc_tokens, acc_nodes, bonus)."""
    acc_t, acc_n = [], []
    cur = -1
    while True:
        want = int(y[0 if cur < 0 else cur + 1])
        nxt = -1
        for c, p in enumerate(parent):
            if int(p) == cur and int(token[c]) == want:
                nxt = c
                break
        if nxt < 0:
            break
        acc_t.append(int(token[nxt]))
        acc_n.append(nxt)
        cur = nxt
    return acc_t, acc_n, int(y[0 if cur < 0 else cur + 1])


@dataclass
class Session:
    """One user's server-side state: the committed context's KV (all but the last committed
    token, amb. A2) and the last committed token (the next root)."""
    cache: Cache
    last_token: int
    session_id: int
    round: int = 0

    @property
    def context_len(self):
        return len(self.cache) + 1


@dataclass
class Request:
    session: Session
    parent: np.ndarray
    token: np.ndarray
    context_len: int = -1       # -1: use the session's (i.e. valid)
    root_token: int = -1        # -1: use the session's last token
    round: int = -1             # -1: use the session's round counter


@dataclass
class Outcome:
    status: int
    accepted_token: list = field(default_factory=list)
    accepted_node: list = field(default_factory=list)
    bonus: int = -1
    row_target: np.ndarray = None   # y per slot
    row_score: np.ndarray = None    # top-1 score per slot
    logits: np.ndarray = None       # [S, V]
    tree_k: list = None
    tree_v: list = None

    @property
    def accepted_len(self):
        return len(self.accepted_token)


def make_session(W: Weights, prompt, session_id, dense=True):
    """Prefill (prefill is outside the measured path): cache the prompt's first n-1
    tokens; the last prompt token is the first root (amb. A2)."""
    from .model import prefill_dense, decode
    prompt = [int(t) for t in prompt]
    if dense:
        _, cache = prefill_dense(W, prompt[:-1])
    else:
        cache = Cache(W.shape)
        decode(W, cache, prompt[:-1])
    return Session(cache, prompt[-1], session_id)


def commit(session: Session, out: Outcome):
    """O5: append K/V of slot 0 and of the accepted nodes' slots, in path order; next root = bonus."""
    slots = [0] + [n + 1 for n in out.accepted_node]
    for l in range(session.cache.shape.n_layers):
        session.cache.append(l, out.tree_k[l][slots], out.tree_v[l][slots])
    session.last_token = out.bonus
    session.round += 1


def verify_one(W: Weights, req: Request, mode="greedy", temperature=0.0, seed=0, keep_logits=True):
    return verify_batch(W, [req], mode, temperature, seed, auto_commit=False, keep_logits=keep_logits)[0]


def verify_batch(W: Weights, reqs, mode="greedy", temperature=0.0, seed=0, auto_commit=True,
                 keep_logits=True):
    """A batch is a list of independent requests: no request reads another's state (amb. A4,
    A17), so the batch result is by construction the list of solo results.  The LM head
    is applied to all requests' rows in one pass over the vocabulary (same arithmetic per row)."""
    s = W.shape
    staged = []
    for req in reqs:
        ses = req.session
        root = ses.last_token if req.root_token < 0 else req.root_token
        ctx = ses.context_len if req.context_len < 0 else req.context_len
        rnd = ses.round if req.round < 0 else req.round
        parent = [int(p) for p in req.parent]
        token = [int(t) for t in req.token]
        st = validate(parent, token, root, s.vocab, ctx, len(ses.cache))
        if st != OK:
            staged.append((st, None))
            continue
        hf, tk, tv = tree_forward(W, ses.cache, root, parent, token)
        staged.append((st, (parent, token, rnd, ses.session_id, hf, tk, tv)))
    rows = [x[1][4] for x in staged if x[0] == OK]
    logits_all = lm_logits(W, np.concatenate(rows)) if rows else None
    outs, off = [], 0
    for st, x in staged:
        if st != OK:
            outs.append(Outcome(status=st))
            continue
        parent, token, rnd, sid, hf, tk, tv = x
        logits = logits_all[off:off + hf.shape[0]]
        off += hf.shape[0]
        scores = target_scores(logits, mode, temperature, seed, rnd, sid)
        y = argmax_lowest(scores)
        acc_t, acc_n, bonus = walk(parent, token, y)
        outs.append(Outcome(OK, acc_t, acc_n, bonus, y, scores.max(axis=-1),
                            logits if keep_logits else None, tk, tv))
    if auto_commit:
        for r, o in zip(reqs, outs):
            if o.status == OK:
                commit(r.session, o)
    return outs
