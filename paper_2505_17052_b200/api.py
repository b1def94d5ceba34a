"""Thin Python API over the C ABI.  PyTorch supplies device memory and streams only; every
step of the verify path runs in libspecedge's kernels (no CPU or torch fallback)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class Shape:
    n_layers: int
    d: int
    n_heads: int
    n_kv: int
    head_dim: int
    ffn: int
    vocab: int
    eps: float
    rope_theta: float

    @classmethod
    def of(cls, s):
        return cls(s.n_layers, s.d, s.n_heads, s.n_kv, s.head_dim, s.ffn, s.vocab, s.eps, s.rope_theta)


def tp_unique_id() -> bytes:
    """128-byte NCCL unique id for specedge_model_create_tp (call on one rank, broadcast)."""
    lib = L.load()
    buf = (C.c_uint8 * 128)()
    L.check(lib.specedge_tp_unique_id(C.cast(buf, C.c_void_p)), "tp_unique_id")
    return bytes(buf)


class Model:
    """A target decoder with synthetic weights (Philox(seed), generated on the device)."""

    def __init__(self, shape, weight_seed: int, device: int = 0, max_position: int = 32768,
                 tp_rank: int = 0, tp_size: int = 1, nccl_id: bytes | None = None):
        """tp_size > 1: this process's tensor-parallel shard (include/specedge.h,
        specedge_model_create_tp); every rank passes the same `nccl_id` (see tp_unique_id)."""
        if not torch.cuda.is_available():
            raise RuntimeError("libspecedge needs a CUDA device (sm_100a); no fallback exists")
        self.lib = L.load()
        self.shape = Shape.of(shape)
        self.device = device
        cfg = L.ModelConfig(shape.n_layers, shape.d, shape.n_heads, shape.n_kv, shape.head_dim,
                            shape.ffn, shape.vocab, shape.eps, shape.rope_theta, max_position)
        h = C.c_void_p()
        if tp_size == 1:
            L.check(self.lib.specedge_model_create(C.byref(cfg), C.c_uint64(weight_seed), device, C.byref(h)),
                    "model_create")
        else:
            # nccl_id None: a communicator-less shard (weights / KV introspection only)
            if nccl_id is not None and len(nccl_id) != 128:
                raise ValueError("tp_size > 1 needs the 128-byte NCCL id from tp_unique_id() (or None)")
            idb = None if nccl_id is None else (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
            L.check(self.lib.specedge_model_create_tp(C.byref(cfg), C.c_uint64(weight_seed), device, tp_rank,
                                                      tp_size, None if idb is None else C.cast(idb, C.c_void_p),
                                                      C.byref(h)),
                    "model_create_tp")
        self.h = h
        self.max_position = max_position
        self.tp_rank, self.tp_size = tp_rank, tp_size
        v0, vn = C.c_int32(), C.c_int32()
        L.check(self.lib.specedge_model_tp_info(h, None, None, C.byref(v0), C.byref(vn)), "model_tp_info")
        self.vocab0, self.vocab_n = v0.value, vn.value
        # rank-local head counts (the KV pool of this model stores n_kv_local heads)
        self.n_heads_local = shape.n_heads // tp_size
        self.n_kv_local = shape.n_kv // tp_size

    def tp_fused_enable(self, max_rows: int, stream=None):
        """NEXT-F4: collective (every rank, same max_rows) — fuse the O / down GEMMs with the
        reduce-scatter of their fp32 updates over NVLink peer memory (specedge_tp_fused_enable)."""
        L.check(self.lib.specedge_tp_fused_enable(self.h, max_rows, _stream(stream)), "tp_fused_enable")

    def tp_fused_mode(self) -> str:
        """The reduce-scatter path in effect (include/specedge.h specedge_tp_fused_mode)."""
        return {0: "nccl", 1: "push", 2: "pull", 3: "nvls"}[int(self.lib.specedge_tp_fused_mode(self.h))]

    def close(self):
        if self.h:
            self.lib.specedge_model_destroy(self.h)
            self.h = None

    def weight_rows(self, tensor: int, layer: int, row0: int, nrows: int, cols: int) -> np.ndarray:
        out = np.empty((nrows, cols), np.uint16)
        L.check(self.lib.specedge_debug_weight_rows(self.h, tensor, layer, row0, nrows,
                                                    out.ctypes.data_as(C.c_void_p)), "debug_weight_rows")
        return out

    def workspace(self, max_requests: int, max_rows: int, max_context: int) -> torch.Tensor:
        n = C.c_size_t()
        L.check(self.lib.specedge_workspace_size(self.h, max_requests, max_rows, max_context, C.byref(n)),
                "workspace_size")
        return torch.empty(n.value, dtype=torch.uint8, device=f"cuda:{self.device}")


class KVPool:
    def __init__(self, model: Model, num_pages: int, max_handles: int):
        self.model = model
        self.lib = model.lib
        h = C.c_void_p()
        L.check(self.lib.specedge_kvpool_create(model.h, num_pages, max_handles, C.byref(h)), "kvpool_create")
        self.h = h

    def close(self):
        if self.h:
            self.lib.specedge_kvpool_destroy(self.h)
            self.h = None

    def alloc(self, capacity: int) -> int:
        out = C.c_int32()
        L.check(self.lib.specedge_kv_alloc(self.h, capacity, C.byref(out)), "kv_alloc")
        return out.value

    def free(self, handle: int):
        L.check(self.lib.specedge_kv_free(self.h, handle), "kv_free")

    def set_len(self, handles, lens, stream=None):
        hs = np.ascontiguousarray(handles, np.int32)
        ls = np.ascontiguousarray(lens, np.int32)
        L.check(self.lib.specedge_kv_set_len(self.h, hs.ctypes.data_as(C.c_void_p), ls.ctypes.data_as(C.c_void_p),
                                             len(hs), _stream(stream)), "kv_set_len")

    def get_len(self, handles):
        hs = np.ascontiguousarray(handles, np.int32)
        out = np.empty(len(hs), np.int32)
        L.check(self.lib.specedge_kv_get_len(self.h, hs.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                             len(hs)), "kv_get_len")
        return out

    def fill_random(self, handle: int, n_tokens: int, seed: int, stream_id: int, stream=None):
        L.check(self.lib.specedge_kv_fill_random(self.h, handle, n_tokens, C.c_uint64(seed), stream_id,
                                                 _stream(stream)), "kv_fill_random")

    def prefill(self, handle: int, tokens, ws: torch.Tensor, stream=None):
        t = np.ascontiguousarray(tokens, np.int32)
        L.check(self.lib.specedge_prefill(self.model.h, self.h, handle, t.ctypes.data_as(C.c_void_p), len(t),
                                          _ptr(ws), ws.numel(), _stream(stream)), "prefill")

    def read_kv(self, handle: int, layer: int, kv_sel: int, pos0: int, n: int) -> np.ndarray:
        s = self.model.shape
        out = np.empty((n, self.model.n_kv_local, s.head_dim), np.uint16)
        L.check(self.lib.specedge_debug_read_kv(self.h, handle, layer, kv_sel, pos0, n,
                                                out.ctypes.data_as(C.c_void_p)), "debug_read_kv")
        return out


def pack_trees(trees):
    """CSR packing of draft trees (objects with .n, .parent, .token, .logprob) over requests:
    node_offset[B+1], parent, token (int32) and draft log-prob (float32) — the layout of
    specedge_verify_in (include/specedge.h)."""
    off = np.zeros(len(trees) + 1, np.int32)
    for i, t in enumerate(trees):
        off[i + 1] = off[i] + t.n
    if trees:
        parent = np.concatenate([np.asarray(t.parent) for t in trees]).astype(np.int32)
        token = np.concatenate([np.asarray(t.token) for t in trees]).astype(np.int32)
        logprob = np.concatenate([np.asarray(t.logprob) for t in trees]).astype(np.float32)
    else:
        parent = token = np.zeros(0, np.int32)
        logprob = np.zeros(0, np.float32)
    return off, parent, token, logprob


@dataclass
class Batch:
    """Device-resident verify inputs (specedge_verify_in's arrays) plus host scalars."""
    kv: torch.Tensor
    context_len: torch.Tensor
    root_token: torch.Tensor
    session_id: torch.Tensor
    round: torch.Tensor
    node_offset: torch.Tensor
    parent: torch.Tensor
    token: torch.Tensor
    draft_logprob: torch.Tensor
    total_nodes: int
    max_nodes: int
    max_context_len: int
    draft_q: torch.Tensor | None = None   # [total_nodes, V] fp32, SAMPLE_PQ_DENSE only

    @property
    def num_requests(self):
        return int(self.kv.numel())

    @property
    def rows(self):
        return self.total_nodes + self.num_requests

    @classmethod
    def from_host(cls, kv, context_len, root_token, session_id, rnd, trees, device="cuda",
                  max_context_len=None, max_nodes=None):
        off, parent, token, logprob = pack_trees(trees)
        dev = torch.device(device)
        t32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.int32)).to(dev)
        ctx = np.ascontiguousarray(context_len, np.int32)
        return cls(t32(kv), t32(ctx), t32(root_token),
                   torch.as_tensor(np.ascontiguousarray(session_id, np.uint64).view(np.int64)).to(dev),
                   torch.as_tensor(np.ascontiguousarray(rnd, np.uint32).view(np.int32)).to(dev),
                   t32(off), t32(parent if len(parent) else np.zeros(1, np.int32)),
                   t32(token if len(token) else np.zeros(1, np.int32)),
                   torch.as_tensor(logprob if len(logprob) else np.zeros(1, np.float32)).to(dev),
                   int(off[-1]),
                   int(max_nodes if max_nodes is not None else max([t.n for t in trees] + [0])),
                   int(max_context_len if max_context_len is not None else int(ctx.max())))


@dataclass
class Outputs:
    status: torch.Tensor
    accepted_len: torch.Tensor
    accepted_token: torch.Tensor
    accepted_node: torch.Tensor
    bonus: torch.Tensor
    row_target: torch.Tensor
    row_score: torch.Tensor

    @classmethod
    def alloc(cls, batch: Batch, device="cuda"):
        B, T, R = batch.num_requests, max(1, batch.total_nodes), batch.rows
        z = lambda n, dt=torch.int32: torch.full((n,), -7, dtype=dt, device=device)
        return cls(z(B), z(B), z(T), z(T), z(B), z(R), torch.zeros(R, dtype=torch.float32, device=device))


def _vin(batch: Batch, mode, temperature, seed, auto_commit):
    return L.VerifyIn(batch.num_requests, batch.total_nodes, batch.max_nodes, batch.max_context_len, mode,
                      float(temperature), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF).value, int(auto_commit),
                      batch.kv.data_ptr(), batch.context_len.data_ptr(), batch.root_token.data_ptr(),
                      batch.session_id.data_ptr(), batch.round.data_ptr(), batch.node_offset.data_ptr(),
                      batch.parent.data_ptr(), batch.token.data_ptr(), batch.draft_logprob.data_ptr(),
                      None if batch.draft_q is None else batch.draft_q.data_ptr())


def _vout(o: Outputs):
    return L.VerifyOut(o.status.data_ptr(), o.accepted_len.data_ptr(), o.accepted_token.data_ptr(),
                       o.accepted_node.data_ptr(), o.bonus.data_ptr(),
                       None if o.row_target is None else o.row_target.data_ptr(),
                       None if o.row_score is None else o.row_score.data_ptr())


def verify(model: Model, pool: KVPool, batch: Batch, ws: torch.Tensor, mode=L.GREEDY, temperature=0.0, seed=0,
           auto_commit=True, out: Outputs | None = None, stream=None) -> Outputs:
    out = out if out is not None else Outputs.alloc(batch, batch.kv.device)
    vin, vout = _vin(batch, mode, temperature, seed, auto_commit), _vout(out)
    L.check(model.lib.specedge_verify_batch(model.h, pool.h, C.byref(vin), C.byref(vout), _ptr(ws), ws.numel(),
                                            _stream(stream)), "verify_batch")
    return out


def kv_commit(model: Model, pool: KVPool, batch: Batch, out: Outputs, ws: torch.Tensor, stream=None):
    vin, vout = _vin(batch, L.GREEDY, 0.0, 0, True), _vout(out)
    L.check(model.lib.specedge_kv_commit(model.h, pool.h, C.byref(vin), C.byref(vout), _ptr(ws), ws.numel(),
                                         _stream(stream)), "kv_commit")


@dataclass
class HostBatch:
    """Pinned host copies of a Batch's arrays for the end-to-end entry point."""
    arrays: dict
    total_nodes: int
    max_nodes: int
    max_context_len: int
    num_requests: int

    @classmethod
    def of(cls, b: Batch):
        a = {k: getattr(b, k).cpu().pin_memory() for k in
             ("kv", "context_len", "root_token", "session_id", "round", "node_offset", "parent", "token",
              "draft_logprob")}
        return cls(a, b.total_nodes, b.max_nodes, b.max_context_len, b.num_requests)

    def nbytes(self):
        return sum(t.numel() * t.element_size() for k, t in self.arrays.items() if k != "draft_logprob")


def verify_host(model: Model, pool: KVPool, hb: HostBatch, ws: torch.Tensor, outs: dict, mode=L.GREEDY,
                temperature=0.0, seed=0, auto_commit=True, stream=None):
    a = hb.arrays
    vin = L.VerifyIn(hb.num_requests, hb.total_nodes, hb.max_nodes, hb.max_context_len, mode, float(temperature),
                     seed, int(auto_commit), a["kv"].data_ptr(), a["context_len"].data_ptr(),
                     a["root_token"].data_ptr(), a["session_id"].data_ptr(), a["round"].data_ptr(),
                     a["node_offset"].data_ptr(), a["parent"].data_ptr(), a["token"].data_ptr(),
                     a["draft_logprob"].data_ptr(), None)
    vout = L.VerifyOut(*(outs[k].data_ptr() for k in ("status", "accepted_len", "accepted_token",
                                                      "accepted_node", "bonus", "row_target", "row_score")))
    L.check(model.lib.specedge_verify_batch_host(model.h, pool.h, C.byref(vin), C.byref(vout), _ptr(ws),
                                                 ws.numel(), _stream(stream)), "verify_batch_host")


def host_outputs(hb: HostBatch):
    B, T, R = hb.num_requests, max(1, hb.total_nodes), hb.total_nodes + hb.num_requests
    z = lambda n, dt=torch.int32: torch.zeros(n, dtype=dt).pin_memory()
    return dict(status=z(B), accepted_len=z(B), accepted_token=z(T), accepted_node=z(T), bonus=z(B),
                row_target=z(R), row_score=z(R, torch.float32))


def graph_stats(model: Model, reset: bool = False) -> dict:
    """Verify-step CUDA-graph cache counters (include/specedge.h specedge_graph_stats)."""
    out = (C.c_int64 * 3)()
    L.check(model.lib.specedge_graph_stats(model.h, C.cast(out, C.c_void_p), 1 if reset else 0), "graph_stats")
    return dict(replays=out[0], captures=out[1], plain=out[2])


def last_launch_count() -> int:
    return int(L.load().specedge_last_launch_count())


def debug_read_tree_kv(model: Model, ws: torch.Tensor, batch: Batch, layer: int, kv_sel: int, row0: int,
                       n: int) -> np.ndarray:
    """Tree K/V scratch rows [row0, row0+n) of the last verify of `batch` with workspace `ws`, as
    fp16 bits [n][n_kv][head_dim] (test introspection)."""
    out = np.empty((n, model.n_kv_local, model.shape.head_dim), np.uint16)
    L.check(model.lib.specedge_debug_read_tree_kv(model.h, _ptr(ws), ws.numel(), batch.num_requests, batch.rows,
                                                  layer, kv_sel, row0, n, out.ctypes.data_as(C.c_void_p)),
            "debug_read_tree_kv")
    return out


def debug_gemm(W: torch.Tensor, X: torch.Tensor, stream=None) -> torch.Tensor:
    """out[r][m] = sum_k X[r,k] W[m,k] through the tcgen05 GEMM kernel (fp32 out)."""
    M, K = W.shape
    R = X.shape[0]
    out = torch.empty((R, M), dtype=torch.float32, device=W.device)
    L.check(L.load().specedge_debug_gemm(_ptr(W), _ptr(X), _ptr(out), M, R, K, _stream(stream)), "debug_gemm")
    return out


def debug_attention(q, k_prefix, v_prefix, k_tree, v_tree, anc, n_splits=1, stream=None):
    """q [S][G][hd] bf16; prefix [L][hd]; tree [S][hd]; anc [S-1] int64 (uint64 bits)."""
    S, G, hd = q.shape
    Lc = 0 if k_prefix is None else k_prefix.shape[0]
    o = torch.empty((S, G, hd), dtype=torch.float32, device=q.device)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device=q.device)
    L.check(L.load().specedge_debug_attention(_ptr(q), _ptr(k_prefix), _ptr(v_prefix), _ptr(k_tree), _ptr(v_tree),
                                              _ptr(anc), S, G, hd, Lc, n_splits, _ptr(o), _ptr(ws), ws.numel(),
                                              _stream(stream)), "debug_attention")
    return o


def debug_last_logits(model: Model, ws: torch.Tensor, batch: Batch, stream=None) -> torch.Tensor:
    """fp32 logits of the last verify's rows over this rank's vocab shard
    [model.vocab0, model.vocab0 + model.vocab_n) (all of V when tp_size == 1)."""
    out = torch.empty((batch.rows, model.vocab_n), dtype=torch.float32, device=ws.device)
    L.check(model.lib.specedge_debug_last_logits(model.h, _ptr(ws), ws.numel(), batch.num_requests, batch.rows,
                                                 _ptr(out), _stream(stream)), "debug_last_logits")
    return out


class Scheduler:
    """NEXT-F1 pipeline-aware verification scheduler (include/specedge.h; host only, no GPU)."""

    def __init__(self, capacity: int, ewma_weight: float = 0.2, fixed_depth: int = 0, init_verify_ms: float = 0.0,
                 init_draft_pass_ms: float = 0.0, init_rtt_ms: float = 0.0):
        self.lib = L.load()
        cfg = L.SchedulerConfig(capacity, ewma_weight, fixed_depth, init_verify_ms, init_draft_pass_ms, init_rtt_ms)
        h = C.c_void_p()
        L.check(self.lib.specedge_scheduler_create(C.byref(cfg), C.byref(h)), "scheduler_create")
        self.h = h
        self.capacity = capacity

    def close(self):
        if self.h:
            self.lib.specedge_scheduler_destroy(self.h)
            self.h = None

    def admit(self, session_id: int, kv_handle: int, length: int, arrival_ms: float) -> bool:
        """False on a protocol error (the session already has an outstanding request)."""
        r = L.SchedRequest(session_id, kv_handle, length, arrival_ms)
        st = self.lib.specedge_scheduler_admit(self.h, C.byref(r))
        if st == L.E_PROTOCOL:
            return False
        L.check(st, "scheduler_admit")
        return True

    def plan(self):
        """-> (list of (session_id, kv_handle, length, arrival_ms), padded_len); ([], 0) if idle."""
        buf = (L.SchedRequest * self.capacity)()
        n, pad = C.c_int32(), C.c_int32()
        L.check(self.lib.specedge_scheduler_plan(self.h, C.cast(buf, C.c_void_p), self.capacity, C.byref(n),
                                                 C.byref(pad)), "scheduler_plan")
        return [(buf[i].session_id, buf[i].kv_handle, buf[i].length, buf[i].arrival_ms) for i in range(n.value)], \
            pad.value

    def complete(self, sessions, verify_ms: float):
        arr = (C.c_uint64 * max(1, len(sessions)))(*sessions)
        L.check(self.lib.specedge_scheduler_complete(self.h, C.cast(arr, C.c_void_p), len(sessions), verify_ms),
                "scheduler_complete")

    def observe(self, kind: int, ms: float):
        L.check(self.lib.specedge_scheduler_observe(self.h, kind, ms), "scheduler_observe")

    def state(self):
        d, q, o = C.c_int32(), C.c_int32(), C.c_int32()
        est = (C.c_double * 3)()
        L.check(self.lib.specedge_scheduler_state(self.h, C.byref(d), C.byref(q), C.byref(o),
                                                  C.cast(est, C.c_void_p)), "scheduler_state")
        return dict(depth=d.value, queued=q.value, outstanding=o.value, estimates=list(est))


def calibrate_draft_depth(verify_ms: float, draft_pass_ms: float, rtt_ms: float) -> int:
    return int(L.load().specedge_calibrate_draft_depth(verify_ms, draft_pass_ms, rtt_ms))


def draft_tree(model: Model, pool: KVPool, handle: int, context_len: int, root_token: int, session_id: int,
               budget: int, depth: int, branching: int, ws: torch.Tensor, head=(), stream=None):
    """NEXT-F3: build a draft tree with this model as the draft model (include/specedge.h,
    specedge_draft_tree); `head` (tokens below the root) = proactive expansion under that path.
    Returns (parent, token, logprob) numpy arrays."""
    parent = np.zeros(budget, np.int32)
    token = np.zeros(budget, np.int32)
    logprob = np.zeros(budget, np.float32)
    n = C.c_int32()
    hd = np.ascontiguousarray(head, np.int32) if len(head) else None
    L.check(model.lib.specedge_draft_tree(model.h, pool.h, handle, context_len, root_token,
                                          C.c_uint64(session_id & 0xFFFFFFFFFFFFFFFF).value,
                                          None if hd is None else hd.ctypes.data_as(C.c_void_p),
                                          0 if hd is None else len(hd), budget, depth,
                                          branching, _ptr(ws), ws.numel(), _stream(stream),
                                          parent.ctypes.data_as(C.c_void_p), token.ctypes.data_as(C.c_void_p),
                                          logprob.ctypes.data_as(C.c_void_p), C.byref(n)), "draft_tree")
    k = n.value
    return parent[:k], token[:k], logprob[:k]
