"""Acceptance planting (setup-time input shaping, SURVEY.md §8(d) "Acceptance planting").

The driver is verifier-agnostic: it is handed a callable `targets(trees) -> list[np.ndarray]`
that returns, per request, the target token y[slot] for every slot (slot 0 = root, slot i+1 =
node i).  It never computes anything of the method itself.  Parity tests plant with the oracle;
the benchmark plants with the library under test (the benchmark is not a parity check).

Procedure for a request with planted length a:
  1. pick the max-cumulative-logprob path n_1..n_a of depth a;
  2. for k = 1..a: query targets, set token(n_k) = y[slot(parent(n_k))]; if a sibling already
     holds that token, swap the two tokens (keeps siblings distinct);
  3. finally re-draw any child of n_a whose token equals y[slot(n_a)].
Changing token(n_k) only changes targets at n_k's subtree, so earlier levels stay matched.
"""
from __future__ import annotations

import numpy as np

from .trees import Tree, best_path


def draw_accept_lengths(rng: np.random.Generator, trees: list[Tree], mu: float, sigma: float):
    """a_r = clip(round(N(mu - 1, sigma)), 0, depth_max) (tokens/verify = a + 1)."""
    out = []
    for t in trees:
        dmax = int(t.depth().max()) if t.n else 0
        a = int(np.clip(np.rint(rng.normal(mu - 1.0, sigma)), 0, dmax))
        out.append(a)
    return out


def draw_accept_lengths_at_mean(rng: np.random.Generator, trees: list[Tree], mu: float, sigma: float):
    """draw_accept_lengths, then the batch total moved to round((mu - 1) * B) (the bench's workload:
    every request set, on every rank, verifies the profile mean mu of Table 1 per request, P:375-385,
    instead of whatever its random draw gave): the largest lengths are lowered / the smallest raised,
    one token at a time, within [0, depth_max]."""
    a = draw_accept_lengths(rng, trees, mu, sigma)
    dmax = [int(t.depth().max()) if t.n else 0 for t in trees]
    target = int(round((mu - 1.0) * len(trees)))
    while sum(a) > target and any(x > 0 for x in a):
        i = max(range(len(a)), key=lambda j: (a[j], -j))
        a[i] -= 1
    while sum(a) < target and any(x < d for x, d in zip(a, dmax)):
        i = min((j for j in range(len(a)) if a[j] < dmax[j]), key=lambda j: (a[j], j))
        a[i] += 1
    return a


def plant(trees: list[Tree], targets, accept_len: list[int], vocab: int,
          rng: np.random.Generator) -> list[Tree]:
    trees = [t.copy() for t in trees]
    paths = [best_path(t, a) for t, a in zip(trees, accept_len)]
    kmax = max([len(p) for p in paths] + [0])
    for k in range(kmax):
        y = targets(trees)
        for r, (t, path) in enumerate(zip(trees, paths)):
            if k >= len(path):
                continue
            node = path[k]
            par = int(t.parent[node])
            want = int(y[r][0 if par < 0 else par + 1])
            if int(t.token[node]) == want:
                continue
            for s in range(t.n):
                if s != node and int(t.parent[s]) == par and int(t.token[s]) == want:
                    t.token[s] = t.token[node]
                    break
            t.token[node] = want
    y = targets(trees)
    for r, (t, path) in enumerate(zip(trees, paths)):
        stop = -1 if not path else path[-1]
        want = int(y[r][0 if stop < 0 else stop + 1])
        kids = [c for c in range(t.n) if int(t.parent[c]) == stop]
        used = {int(t.token[c]) for c in kids}
        for c in kids:
            if int(t.token[c]) == want:
                while True:
                    nt = int(rng.integers(0, vocab))
                    if nt != want and nt not in used:
                        break
                used.discard(int(t.token[c]))
                used.add(nt)
                t.token[c] = nt
    return trees
