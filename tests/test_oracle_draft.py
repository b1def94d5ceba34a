"""Pins of the NEXT-F3 oracle (oracle/draft.py: pooled top-budget draft-tree construction, best
path; App. A):
  * S:126's worked example (table q = [0.5, 0.25, 0.125, 0.125], budget 3, branching 2, depth 2 ->
    nodes "0" -0.693, "1" -1.386, "0->0" -1.386) and S:134's best path [0, 0] (deeper leaf wins);
  * branching 1, budget = depth = k is repeated greedy decoding (Appendix B chain mode);
  * structural invariants on random context-dependent tables: <= budget nodes, parents precede
    children, ancestor closure, distinct sibling tokens, cum = parent cum + logprob, depth <= passes;
  * the kept set after every pass is exactly the top-budget of the pooled candidates in the order
    (-cum, depth, token), checked against a brute-force re-sort."""
import math

import numpy as np

from oracle import draft as OD


def test_spec_worked_example_and_best_path():
    q = np.log(np.array([0.5, 0.25, 0.125, 0.125]))
    parent, token, lp, cum = OD.build_draft_tree(lambda path: q, budget=3, depth=2, branching=2)
    assert token == [0, 1, 0] and parent == [-1, -1, 0]
    np.testing.assert_allclose(cum, [-math.log(2), -math.log(4), -math.log(4)], atol=1e-12)
    assert [token[i] for i in OD.best_path(parent, token, cum)] == [0, 0]


def test_branching_one_is_greedy_decoding():
    rng = np.random.default_rng(2)
    tables = {}

    def lp(path):
        if path not in tables:
            tables[path] = np.log(rng.dirichlet(np.ones(9)))
        return tables[path]
    parent, token, _, _ = OD.build_draft_tree(lp, budget=5, depth=5, branching=1)
    greedy, path = [], ()
    for _ in range(5):
        t = int(np.argmax(lp(path)))
        greedy.append(t)
        path = path + (t,)
    assert token == greedy and parent == [-1, 0, 1, 2, 3]


def test_invariants_and_pooled_top_budget():
    rng = np.random.default_rng(7)
    for trial in range(30):
        V = int(rng.integers(3, 12))
        tables = {}

        def lp(path):
            if path not in tables:
                tables[path] = np.log(rng.dirichlet(np.full(V, 0.5)))
            return tables[path]
        budget, depth, b = int(rng.integers(1, 20)), int(rng.integers(1, 6)), int(rng.integers(1, min(V, 4) + 1))
        passes = []
        parent, token, lps, cum = OD.build_draft_tree(lp, budget, depth, b, passes_out=passes)
        n = len(parent)
        assert n <= budget
        depths = []
        for i in range(n):
            assert -1 <= parent[i] < i
            depths.append(1 if parent[i] < 0 else depths[parent[i]] + 1)
            base = 0.0 if parent[i] < 0 else cum[parent[i]]
            assert abs(cum[i] - (base + lps[i])) < 1e-9
            path, j = [], i
            while j >= 0:
                path.append(token[j])
                j = parent[j]
            assert abs(lps[i] - lp(tuple(path[::-1][:-1]))[token[i]]) < 1e-12
        assert max(depths + [0]) <= depth
        sib = {}
        for i in range(n):
            assert token[i] not in sib.setdefault(parent[i], set())
            sib[parent[i]].add(token[i])
        # brute force: rebuild every pass from its pooled candidates and re-sort
        kept = []   # list of (path tuple)
        frontier_paths = [()]
        for ps in passes:
            cand = [(p_, 0) for p_ in kept]
            for fp in frontier_paths:
                for t in np.argsort(-lp(fp), kind="stable")[:b]:
                    cand.append((fp + (int(t),), 1))
            def key(c):
                pth = c[0]
                cm = sum(lp(pth[:k])[pth[k]] for k in range(len(pth)))
                return (-cm, len(pth), pth[-1])
            top = sorted(cand, key=key)[:budget]
            top_paths = set(c[0] for c in top)
            # reconstruct the oracle's kept paths of this pass
            pth = []
            for i, (pp, tt) in enumerate(ps):
                pth.append((() if pp < 0 else pth[pp]) + (tt,))
            got_paths = set(pth)
            assert got_paths == top_paths, trial
            frontier_paths = [c[0] for c in top if c[1] == 1]
            kept = [c[0] for c in top]
