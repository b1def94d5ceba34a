"""NEXT-F3 on the GPU: specedge_draft_tree (the edge's pooled top-budget draft-tree builder on the
verify kernels) against oracle/draft.py with the oracle's own draft model (oracle/model.py) on the
same seeded weights and contexts.  Trees must be identical (parents, tokens) and log-probs within
LP_TOL = 2 x north_star's logit tolerance (a log-prob is a logit minus a log-sum-exp, each within
2e-2), unless a decision of the oracle sits within that tolerance (a top-`branching` cut or the
budget cut closer than 2 * LP_TOL): counted as exempt.  No bound uses the library's own error."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import draft as OD  # noqa: E402
from oracle import verify as OV  # noqa: E402
from oracle.model import Weights  # noqa: E402
from synth.configs import TINY, SMALL128  # noqa: E402
from tests.gpu_helpers import LOGIT_TOL  # noqa: E402

LP_TOL = 2 * LOGIT_TOL


@pytest.fixture(scope="module")
def api():
    from paper_2505_17052_b200 import api as A
    return A


def _margins(lp_fn, passes, b, budget):
    """Smallest decision margin of the oracle build: top-b cut per proposal and the budget cut."""
    m = np.inf
    kept, frontier = [], [()]
    for ps in passes:
        cand = list(kept)
        for fp in frontier:
            l = np.sort(lp_fn(fp))[::-1]
            if len(l) > b:
                m = min(m, l[b - 1] - l[b])
            order = np.argsort(-lp_fn(fp), kind="stable")[:b]
            cand += [fp + (int(t),) for t in order]
        cums = sorted([sum(lp_fn(p[:k])[p[k]] for k in range(len(p))) for p in cand], reverse=True)
        if len(cums) > budget:
            m = min(m, cums[budget - 1] - cums[budget])
        pth = []
        for (pp, tt) in ps:
            pth.append((() if pp < 0 else pth[pp]) + (tt,))
        frontier = [p for p in pth if p not in kept]
        kept = pth
    return m


@pytest.mark.parametrize("shape,budget,depth,branching", [(TINY, 8, 4, 3), (TINY, 32, 7, 4), (SMALL128, 16, 5, 2),
                                                          (TINY, 5, 5, 1)])
def test_draft_tree_matches_oracle(api, shape, budget, depth, branching):
    rng = np.random.default_rng(budget + depth)
    W = Weights(shape, 11)
    prompts = [[int(t) for t in rng.integers(0, shape.vocab, n)] for n in (23, 40)]
    model = api.Model(shape, 11, max_position=4096)
    try:
        pool = api.KVPool(model, 16, 4)
        ws = model.workspace(1, budget + 1, 256)
        kinds = []
        for i, p in enumerate(prompts):
            ses = OV.make_session(W, p, 70 + i)
            h = pool.alloc(200)
            pool.prefill(h, p, ws)
            lp_fn = OD.model_lp(W, ses)
            passes = []
            o_par, o_tok, o_lp, o_cum = OD.build_draft_tree(lp_fn, budget, depth, branching, passes_out=passes)
            g_par, g_tok, g_lp = api.draft_tree(model, pool, h, ses.context_len, ses.last_token, ses.session_id,
                                                budget, depth, branching, ws)
            same = list(g_par) == o_par and list(g_tok) == o_tok
            if same:
                assert np.abs(np.asarray(g_lp, np.float64) - np.asarray(o_lp)).max() <= LP_TOL
                kinds.append("exact")
            else:
                margin = _margins(lp_fn, passes, branching, budget)
                assert margin <= 2 * LP_TOL, (margin, list(g_tok), o_tok, list(g_par), o_par)
                kinds.append("exempt")
            # the builder never commits: the cache is unchanged
            assert int(pool.get_len([h])[0]) == len(ses.cache)
        assert len(kinds) == len(prompts)
        pool.close()
    finally:
        model.close()


@pytest.mark.parametrize("shape", [TINY, SMALL128])
def test_proactive_expansion_matches_oracle(api, shape):
    """§4.2 proactive drafting: the subtree drafted under the best path's leaf (oracle best_path of
    the oracle tree) equals the oracle's proactive_expand."""
    rng = np.random.default_rng(31)
    W = Weights(shape, 11)
    p = [int(t) for t in rng.integers(0, shape.vocab, 30)]
    model = api.Model(shape, 11, max_position=4096)
    try:
        pool = api.KVPool(model, 16, 4)
        ws = model.workspace(1, 40, 256)
        ses = OV.make_session(W, p, 90)
        h = pool.alloc(200)
        pool.prefill(h, p, ws)
        lp_fn = OD.model_lp(W, ses)
        par, tok, _, cum = OD.build_draft_tree(lp_fn, 12, 4, 3)
        head = [tok[i] for i in OD.best_path(par, tok, cum)]
        passes = []
        o_par, o_tok, o_lp, _ = OD.build_draft_tree(lambda path: lp_fn(tuple(head) + tuple(path)), 10, 3, 2,
                                                     passes_out=passes)
        assert (o_par, o_tok) == tuple(list(x) for x in OD.proactive_expand(lp_fn, head, 10, 3, 2)[:2])
        g_par, g_tok, g_lp = api.draft_tree(model, pool, h, ses.context_len, ses.last_token, ses.session_id,
                                            10, 3, 2, ws, head=head)
        if list(g_par) == o_par and list(g_tok) == o_tok:
            assert np.abs(np.asarray(g_lp, np.float64) - np.asarray(o_lp)).max() <= LP_TOL
        else:
            margin = _margins(lambda path: lp_fn(tuple(head) + tuple(path)), passes, 2, 10)
            assert margin <= 2 * LP_TOL, (margin, list(g_tok), o_tok)
        pool.close()
    finally:
        model.close()
