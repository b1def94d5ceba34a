"""NEXT-F2 on the GPU: SAMPLE_PQ_DENSE (dense-q speculative sampling of sampled draft chains,
PAPER.md App. B; include/specedge.h) against the oracle (oracle/pq.py) on the same seeded inputs.

The chains are sampled the way an edge would: at slot i the draft distribution is
q_i = mix * p_i + (1 - mix) * Dirichlet noise (p_i = the oracle's target distribution given the
chain so far, so acceptance is neither certain nor hopeless) and x_i ~ q_i.  Outcomes (accepted
nodes, bonus) must equal the oracle's exactly, except where a decision is within what the logit
tolerance asserted on the same run's logits (eps = 2e-2 or the oracle-derived bound) allows: |u - p/q| <= 4 eps/T * p/q
(accept test) or a residual Gumbel-max margin below the propagated bound — counted as exempt
(SURVEY amb. A21 reading, DESIGN.md R-pq).  The bound never uses the library's measured error."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pq as OPQ  # noqa: E402
from oracle import verify as OV  # noqa: E402
from oracle.model import Weights, lm_logits, tree_forward  # noqa: E402
from synth.configs import TINY, SMALL128  # noqa: E402
from synth.trees import Tree  # noqa: E402
from tests.gpu_helpers import check_logits, oracle_noise_floor  # noqa: E402


@pytest.fixture(scope="module")
def api():
    from paper_2505_17052_b200 import api as A
    return A


def _sample_chain(W, session, n, T, rng, mix):
    """Edge-side sampling of a chain of n tokens with explicit draft rows q_i."""
    invT = OV.inv_temperature(T)
    toks, qs = [], []
    for i in range(n):
        parent = list(range(-1, i - 1))
        hf, _, _ = tree_forward(W, session.cache, session.last_token, parent, toks)
        p = OPQ.softmax_t(lm_logits(W, hf[-1:])[0], invT)
        q = mix * p + (1 - mix) * rng.dirichlet(np.full(W.shape.vocab, 0.3))
        q = (q / q.sum()).astype(np.float32).astype(np.float64)
        q /= q.sum()
        x = int(rng.choice(W.shape.vocab, p=q))
        toks.append(x)
        qs.append(q.astype(np.float32))
    return Tree(np.arange(-1, n - 1, dtype=np.int32), np.asarray(toks, np.int32), np.zeros(n, np.float32)), \
        np.stack(qs) if n else np.zeros((0, W.shape.vocab), np.float32)


def _compare(o, g, r, noff, eps, T, q_rows, gumbel_fn):
    """'exact' or 'exempt' (decision within the error bound), else raise."""
    a = int(g["accepted_len"][r])
    got_nodes = list(g["accepted_node"][noff[r]:noff[r] + a])
    if a == len(o.accepted_node) and got_nodes == o.accepted_node and int(g["bonus"][r]) == o.bonus:
        return "exact"
    rel = 4.0 * eps / T
    # accept decisions up to the first divergence
    for i, (u, ratio) in enumerate(zip(o.uniforms, o.ratios)):
        if abs(u - ratio) <= rel * ratio + 1e-6:
            return "exempt"
        if i >= min(a, len(o.accepted_node)):
            break
    # same accepted path, different bonus: residual / leaf Gumbel-max margin
    stop = o.stop
    p = o.p_rows[stop]
    if stop < len(o.ratios):
        resid = np.maximum(0.0, p - q_rows[stop])
        with np.errstate(divide="ignore"):
            sc = np.where(resid > 0, np.log(np.where(resid > 0, resid, 1)) + gumbel_fn(stop), -np.inf)
        bound = np.where(resid > 0, rel * p / np.maximum(resid, 1e-300), np.inf)
    else:
        sc = np.log(np.maximum(p, 1e-300)) + gumbel_fn(stop)
        bound = np.full_like(sc, rel)
    b_or, b_g = o.bonus, int(g["bonus"][r])
    if b_g >= 0 and sc[b_or] - sc[b_g] <= bound[b_or] + bound[b_g]:
        return "exempt"
    raise AssertionError(f"request {r}: gpu (a={a}, bonus={b_g}, nodes={got_nodes}) != oracle "
                         f"(a={len(o.accepted_node)}, bonus={b_or}, nodes={o.accepted_node}); ratios "
                         f"{o.ratios}, u {o.uniforms}")


@pytest.mark.parametrize("shape,T,mix", [(TINY, 1.0, 0.8), (TINY, 0.7, 0.5), (SMALL128, 1.0, 0.9)])
def test_pq_dense_matches_oracle(api, shape, T, mix):
    rng = np.random.default_rng(int(T * 10) + shape.d)
    B = 6
    prompts = [[int(t) for t in rng.integers(0, shape.vocab, n)] for n in (20, 33, 9, 40, 17, 28)]
    W = Weights(shape, 3)
    sessions = [OV.make_session(W, p, 500 + i) for i, p in enumerate(prompts)]
    for i, s in enumerate(sessions):
        s.round = 7 + i
    trees, qrows = [], []
    for i, n in enumerate((6, 8, 1, 0, 8, 5)):
        t, q = _sample_chain(W, sessions[i], n, T, rng, mix)
        trees.append(t)
        qrows.append(q)
    seed = 4242
    refs = OPQ.verify_pq(W, [OV.Request(s, t.parent, t.token) for s, t in zip(sessions, trees)], qrows, T, seed,
                         auto_commit=False)
    model = api.Model(shape, 3, max_position=4096)
    try:
        cap = max(len(p) for p in prompts) + 64
        pool = api.KVPool(model, ((cap + 63) // 64) * B + 4, B + 2)
        ws = model.workspace(B, B * 65, cap)
        handles = []
        for p in prompts:
            h = pool.alloc(cap)
            pool.prefill(h, p, ws)
            handles.append(h)
        batch = api.Batch.from_host(handles, [s.context_len for s in sessions], [s.last_token for s in sessions],
                                    [s.session_id for s in sessions], [s.round for s in sessions], trees,
                                    max_context_len=cap)
        batch.draft_q = torch.from_numpy(np.concatenate(qrows).astype(np.float32)).cuda()
        out = api.verify(model, pool, batch, ws, mode=api.L.SAMPLE_PQ_DENSE, temperature=T, seed=seed,
                         auto_commit=False)
        logits = api.debug_last_logits(model, ws, batch).cpu().numpy()
        torch.cuda.synchronize()
        g = dict(status=out.status.cpu().numpy(), accepted_len=out.accepted_len.cpu().numpy(),
                 accepted_node=out.accepted_node.cpu().numpy(), bonus=out.bonus.cpu().numpy())
        noff = np.cumsum([0] + [t.n for t in trees])
        def run():
            return np.concatenate([o.logits for o in OPQ.verify_pq(
                W, [OV.Request(s, t.parent, t.token) for s, t in zip(sessions, trees)], qrows, T, seed,
                auto_commit=False)])
        bound = check_logits(logits, np.concatenate([o.logits for o in refs]),
                             noise_fn=lambda: oracle_noise_floor(run)[1])
        kinds = []
        for r, o in enumerate(refs):
            assert g["status"][r] == 0
            ses = sessions[r]
            kinds.append(_compare(o, g, r, noff, bound, T, qrows[r],
                                  lambda s, ses=ses: OV.gumbel(seed, ses.round, ses.session_id, s, shape.vocab)))
        assert kinds.count("exempt") <= 1, kinds
        pool.close()
    finally:
        model.close()


def test_pq_dense_rejects_non_chains_and_bad_args(api):
    shape = TINY
    rng = np.random.default_rng(5)
    W = Weights(shape, 3)
    prompts = [[int(t) for t in rng.integers(0, shape.vocab, 12)] for _ in range(2)]
    sessions = [OV.make_session(W, p, 900 + i) for i, p in enumerate(prompts)]
    model = api.Model(shape, 3, max_position=1024)
    try:
        pool = api.KVPool(model, 8, 4)
        ws = model.workspace(2, 2 * 65, 128)
        handles = []
        for p in prompts:
            h = pool.alloc(100)
            pool.prefill(h, p, ws)
            handles.append(h)
        trees = [Tree(np.array([-1, 0, 0], np.int32), np.array([3, 4, 5], np.int32), np.zeros(3, np.float32)),
                 Tree(np.array([-1, 0], np.int32), np.array([6, 7], np.int32), np.zeros(2, np.float32))]
        batch = api.Batch.from_host(handles, [s.context_len for s in sessions], [s.last_token for s in sessions],
                                    [s.session_id for s in sessions], [0, 0], trees, max_context_len=128)
        q = np.full((5, shape.vocab), 1.0 / shape.vocab, np.float32)
        batch.draft_q = torch.from_numpy(q).cuda()
        out = api.verify(model, pool, batch, ws, mode=api.L.SAMPLE_PQ_DENSE, temperature=1.0, seed=1,
                         auto_commit=False)
        st = out.status.cpu().numpy()
        assert st[0] == api.L.REQ_E_UNSUPPORTED and st[1] == 0          # branching tree vs chain
        assert out.bonus.cpu().numpy()[0] == -1
        with pytest.raises(RuntimeError):                                  # T = 0 is not a sampling mode
            api.verify(model, pool, batch, ws, mode=api.L.SAMPLE_PQ_DENSE, temperature=0.0, seed=1)
        batch.draft_q = None
        with pytest.raises(RuntimeError):                                  # dense q rows required
            api.verify(model, pool, batch, ws, mode=api.L.SAMPLE_PQ_DENSE, temperature=1.0, seed=1)
        pool.close()
    finally:
        model.close()
