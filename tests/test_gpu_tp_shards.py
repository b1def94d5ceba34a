"""Tensor-parallel sharding on ONE GPU (SURVEY §8(e) TP regime, P14 "TP = k == TP = 1"): every
shard of specedge_model_create_tp holds, bit for bit, its slice of the tp_size == 1 model —
head-parallel q/k/v rows, the matching Wo input columns, column-parallel gate/up rows, the
matching Wd input columns, the vocab-parallel LM-head rows, replicated embedding and norm gains —
and its KV pool holds its kv heads of the same synthetic cache.  Communicator-less shards
(nccl_id None) make this runnable with one device; the collectives themselves are covered by
tests/test_gpu_tp.py on 2+ GPUs.  Llama-3-70B widths (cfg4; one layer) at TP = 2, 4, 8."""
import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth.configs import LLAMA3_70B, ModelShape  # noqa: E402

SEED = 4
SHAPE = dataclasses.replace(LLAMA3_70B, name="llama3-70b-1l", n_layers=1)
TINY_TP = ModelShape("tiny-tp", 2, 1024, 8, 8, 128, 2048, 1024, 1e-6, 10000.0)


def _rows(model, tensor, layer, idx, cols):
    return np.stack([model.weight_rows(tensor, layer, int(i), 1, cols)[0] for i in idx])


@pytest.fixture(scope="module")
def api():
    from paper_2505_17052_b200 import api as A
    return A


@pytest.mark.parametrize("shape", [TINY_TP, SHAPE], ids=["tiny-tp", "llama3-70b-1l"])
def test_tp_shards_are_slices_of_the_tp1_model(api, shape):
    s = shape
    hd, H, KV, d, F, V = s.head_dim, s.n_heads, s.n_kv, s.d, s.ffn, s.vocab
    rng = np.random.default_rng(5)
    full = api.Model(s, SEED, max_position=256)
    fpool = api.KVPool(full, 4, 2)
    fh = fpool.alloc(128)
    fpool.fill_random(fh, 100, 77, 3)
    try:
        # sampled logical rows / columns of the full model (every row would be ~GBs of host copies)
        pick = lambda n, k: np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, k)]))
        wo_idx, wd_idx = pick(d, 24), pick(d, 24)
        full_wo = _rows(full, 5, 0, wo_idx, H * hd)
        full_wd = _rows(full, 8, 0, wd_idx, F)
        gains = [full.weight_rows(t, 0, 0, 1, d) for t in (10, 11, 12)]
        emb_idx = pick(V, 16)
        emb = _rows(full, 1, 0, emb_idx, d)
        kv_full = [fpool.read_kv(fh, 0, sel, 0, 100) for sel in (0, 1)]
        for tp in (2, 4, 8):
            if KV % tp or H % tp or F % (64 * tp):
                continue
            Hl, KVl, Fl = H // tp, KV // tp, F // tp
            vs = -(-V // tp)
            for rank in range(tp):
                sh = api.Model(s, SEED, max_position=256, tp_rank=rank, tp_size=tp, nccl_id=None)
                spool = api.KVPool(sh, 4, 2)
                try:
                    assert (sh.vocab0, sh.vocab_n) == (rank * vs, min(V, (rank + 1) * vs) - rank * vs)
                    for t, n_loc, off in ((2, Hl * hd, rank * Hl * hd), (3, KVl * hd, rank * KVl * hd),
                                          (4, KVl * hd, rank * KVl * hd), (6, Fl, rank * Fl), (7, Fl, rank * Fl)):
                        loc = pick(n_loc, 8)
                        assert np.array_equal(_rows(sh, t, 0, loc, d), _rows(full, t, 0, loc + off, d)), (tp, rank, t)
                    # row-parallel Wo / Wd: the shard's input columns of every output row
                    wo = _rows(sh, 5, 0, wo_idx, Hl * hd)
                    assert np.array_equal(wo, full_wo[:, rank * Hl * hd:(rank + 1) * Hl * hd]), (tp, rank, "wo")
                    wd = _rows(sh, 8, 0, wd_idx, Fl)
                    assert np.array_equal(wd, full_wd[:, rank * Fl:(rank + 1) * Fl]), (tp, rank, "wd")
                    loc = pick(sh.vocab_n, 8)
                    assert np.array_equal(_rows(sh, 9, 0, loc, d), _rows(full, 9, 0, loc + sh.vocab0, d)), (tp, rank)
                    assert np.array_equal(_rows(sh, 1, 0, emb_idx, d), emb)
                    for t, g in zip((10, 11, 12), gains):
                        assert np.array_equal(sh.weight_rows(t, 0, 0, 1, d), g)
                    # KV pool: this rank's kv heads of the same synthetic cache
                    h = spool.alloc(128)
                    spool.fill_random(h, 100, 77, 3)
                    for sel in (0, 1):
                        assert np.array_equal(spool.read_kv(h, 0, sel, 0, 100),
                                              kv_full[sel][:, rank * KVl:(rank + 1) * KVl]), (tp, rank, sel)
                finally:
                    spool.close()
                    sh.close()
    finally:
        fpool.close()
        full.close()


def test_communicator_less_shard_refuses_to_verify(api):
    sh = api.Model(TINY_TP, SEED, max_position=256, tp_rank=0, tp_size=2, nccl_id=None)
    pool = api.KVPool(sh, 4, 2)
    try:
        from synth.trees import Tree
        h = pool.alloc(64)
        pool.fill_random(h, 9, 1, 0)
        ws = sh.workspace(1, 2, 64)
        tr = Tree(np.array([-1], np.int32), np.array([1], np.int32), np.zeros(1, np.float32))
        b = api.Batch.from_host([h], [10], [3], [1], [0], [tr], max_context_len=64)
        with pytest.raises(RuntimeError, match="status -5"):
            api.verify(sh, pool, b, ws)
    finally:
        pool.close()
        sh.close()
