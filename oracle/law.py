"""The law of (stop node, bonus) under lossless tree verification.

SURVEY §8(c) Lemma / O7: for a fixed tree with distinct sibling tokens, every lossless verifier
that emits a child's token only by descending into that child (P:171 'preserves the exact output
distribution of the server model', citing Leviathan et al.) has
    Pr[stop at v, bonus b] = prod_{w on root->v, w != root} p(tok(w) | parent(w)) * p(b | v)
                             * [b not in tok(children(v))],
with p(. | u) = softmax(l_u / T) the target's next-token distribution at slot u.

O8: the explicit p/q rejection form (children tried in order; accept c with prob p_res(c); on
rejection remove c from p_res and renormalise; if all rejected, bonus ~ p_res) is an
independent formulation; `rejection_law` enumerates it exactly so the tests can pin O7 == O8.
"""
from __future__ import annotations

import numpy as np


def slot_probs(logits, temperature):
    """p(. | slot) = softmax(l / T), float64."""
    z = np.asarray(logits, np.float64) / float(temperature)
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def closed_form_law(parent, token, probs):
    """O7.  probs [S, V].  Returns dict {(stop_slot, bonus): probability}."""
    n = len(parent)
    reach = np.zeros(n + 1)
    reach[0] = 1.0
    for i in range(n):
        ps = 0 if parent[i] < 0 else parent[i] + 1
        reach[i + 1] = reach[ps] * probs[ps, token[i]]
    law = {}
    for s in range(n + 1):
        node = s - 1
        kids = {int(token[c]) for c in range(n) if parent[c] == node}
        for b in range(probs.shape[1]):
            if b not in kids:
                law[(s, b)] = reach[s] * probs[s, b]
    return law


def rejection_law(parent, token, probs, order_key=None):
    """O8 enumerated exactly.  `order_key(c)` orders the children (default: node index)."""
    n = len(parent)
    law: dict = {}

    def visit(slot, mass):
        node = slot - 1
        kids = [c for c in range(n) if parent[c] == node]
        if order_key is not None:
            kids.sort(key=order_key)
        p_res = probs[slot].copy()
        rest = mass
        for c in kids:
            a = p_res[token[c]]
            visit(c + 1, rest * a)
            rest = rest * (1.0 - a)
            p_res[token[c]] = 0.0
            tot = p_res.sum()
            if tot <= 0:
                return
            p_res = p_res / tot
        for b in range(probs.shape[1]):
            if p_res[b] > 0:
                law[(slot, b)] = law.get((slot, b), 0.0) + rest * p_res[b]

    visit(0, 1.0)
    return law
