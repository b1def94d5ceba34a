"""The plain C++ oracle (oracle/cpp/verify_ref.cpp, north_star's "plain, slow CPU C++
implementation") against the numpy oracle, which is itself pinned to the paper and mathematics
(tests/test_oracle_*.py): same seeded weights, caches and trees (prefilled sessions and the
synthetic KV fill, greedy and Gumbel-max sampling) give the same per-slot targets, accepted paths
and bonus tokens, and float64 logits equal up to summation order."""
import numpy as np
import pytest

from oracle import cpp_ref
from oracle import verify as OV
from oracle.model import Cache, Weights, gen_kv_fill
from synth.configs import TINY, SMALL128, ModelShape
from synth.trees import pooled_tree, random_tree

MID = ModelShape("mid", 2, 256, 4, 2, 64, 512, 1000, 1e-5, 500000.0)


@pytest.mark.parametrize("shape", [TINY, MID, SMALL128], ids=lambda s: s.name)
def test_cpp_oracle_equals_numpy_oracle(shape):
    rng = np.random.default_rng(17)
    W = Weights(shape, 9)
    cm = cpp_ref.Model(shape, 9)
    try:
        # a real prefilled session and a synthetic-fill session
        prompt = [int(t) for t in rng.integers(0, shape.vocab, 40)]
        ses = OV.make_session(W, prompt, 123)
        L2 = 70
        c2 = Cache(shape)
        for l in range(shape.n_layers):
            c2.k[l] = gen_kv_fill(55, 3, l, 0, L2, shape.n_kv, shape.head_dim)
            c2.v[l] = gen_kv_fill(55, 3, l, 1, L2, shape.n_kv, shape.head_dim)
        ses2 = OV.Session(c2, int(rng.integers(0, shape.vocab)), 456)
        for mode, T in (("greedy", 0.0), ("sample", 0.8)):
            for tree in (pooled_tree(rng, 12, 4, 3, shape.vocab), random_tree(rng, 9, shape.vocab)):
                for s_, kw in ((ses, dict(cache=(ses.cache.k, ses.cache.v))), (ses2, dict(fill=(55, 3)))):
                    o = OV.verify_one(W, OV.Request(s_, tree.parent, tree.token, round=5), mode, T, 77)
                    c = cm.verify(len(s_.cache), s_.last_token, tree.parent, tree.token, mode=mode, temperature=T,
                                  seed=77, round_=5, session=s_.session_id, want_logits=True, **kw)
                    assert np.abs(c["logits"] - o.logits).max() <= 1e-9 * max(1.0, np.abs(o.logits).max())
                    assert np.array_equal(c["row_target"], o.row_target)
                    assert c["accepted_node"] == o.accepted_node and c["accepted_token"] == o.accepted_token
                    assert c["bonus"] == o.bonus
    finally:
        cm.close()


def test_cpp_oracle_rejects_bad_tree():
    cm = cpp_ref.Model(TINY, 1)
    try:
        with pytest.raises(ValueError):
            cm.verify(5, 1, [-1, 2, 0], [1, 2, 3], fill=(1, 0))
    finally:
        cm.close()
