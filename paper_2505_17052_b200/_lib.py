"""ctypes binding of libspecedge.so (include/specedge.h).  Argument marshalling only: every step
of the verify path runs in the library's CUDA kernels.  There is no fallback: if the shared
library or a CUDA device is missing, construction raises."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPECEDGE_LIB") or os.path.join(HERE, "libspecedge.so")   # env: experiment builds

OK = 0
E_INVALID, E_CUDA, E_OOM, E_WORKSPACE, E_UNSUPPORTED, E_DEVICE, E_PROTOCOL = -1, -2, -3, -4, -5, -6, -7
TIMING_VERIFY, TIMING_DRAFT_PASS, TIMING_RTT = 0, 1, 2
REQ_E_UNSUPPORTED = 8
REQ_OK, REQ_E_TREE, REQ_E_TREE_SIZE, REQ_E_TOKEN, REQ_E_DUP_SIBLING, REQ_E_CONTEXT, \
    REQ_E_KV_CAPACITY, REQ_E_HANDLE = range(8)
GREEDY, SAMPLE_TREE, SAMPLE_PQ_DENSE = 0, 1, 2
MAX_NODES = 64

# every symbol include/specedge.h declares (tests check the .so exports all of them)
EXPORTS = [
    "specedge_model_create", "specedge_model_destroy", "specedge_kvpool_create",
    "specedge_kvpool_destroy", "specedge_kv_alloc", "specedge_kv_free", "specedge_kv_set_len",
    "specedge_kv_get_len", "specedge_kv_fill_random", "specedge_workspace_size", "specedge_prefill",
    "specedge_verify_batch", "specedge_kv_commit", "specedge_verify_batch_host",
    "specedge_debug_weight_rows", "specedge_debug_read_kv", "specedge_debug_read_tree_kv", "specedge_debug_gemm",
    "specedge_debug_last_logits", "specedge_debug_attention", "specedge_last_launch_count",
    "specedge_set_kernel_timing", "specedge_kernel_times", "specedge_tp_unique_id", "specedge_model_create_tp",
    "specedge_model_tp_info", "specedge_calibrate_draft_depth", "specedge_scheduler_create",
    "specedge_scheduler_destroy", "specedge_scheduler_admit", "specedge_scheduler_plan",
    "specedge_scheduler_complete", "specedge_scheduler_observe", "specedge_scheduler_state",
    "specedge_draft_tree", "specedge_tp_fused_enable", "specedge_graph_stats", "specedge_tp_fused_mode",
]
KERNEL_KINDS = ["prep", "embed", "rmsnorm", "gemm_qkv", "attention", "attn_combine", "gemm_o", "gemm_gateup",
                "gemm_down", "gemm_lmhead", "lm_reduce", "walk", "commit", "qkv_rope"]


class ModelConfig(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("eps", C.c_float), ("rope_theta", C.c_double),
                ("max_position", C.c_int32)]


class SchedulerConfig(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("ewma_weight", C.c_double), ("fixed_depth", C.c_int32),
                ("init_verify_ms", C.c_double), ("init_draft_pass_ms", C.c_double), ("init_rtt_ms", C.c_double)]


class SchedRequest(C.Structure):
    _fields_ = [("session_id", C.c_uint64), ("kv_handle", C.c_int32), ("length", C.c_int32),
                ("arrival_ms", C.c_double)]


class VerifyIn(C.Structure):
    _fields_ = [("num_requests", C.c_int32), ("total_nodes", C.c_int32), ("max_nodes", C.c_int32),
                ("max_context_len", C.c_int32), ("mode", C.c_int32), ("temperature", C.c_float),
                ("seed", C.c_uint64), ("auto_commit", C.c_int32),
                ("kv", C.c_void_p), ("context_len", C.c_void_p), ("root_token", C.c_void_p),
                ("session_id", C.c_void_p), ("round", C.c_void_p), ("node_offset", C.c_void_p),
                ("parent", C.c_void_p), ("token", C.c_void_p), ("draft_logprob", C.c_void_p),
                ("draft_q", C.c_void_p)]


class VerifyOut(C.Structure):
    _fields_ = [("status", C.c_void_p), ("accepted_len", C.c_void_p),
                ("accepted_token", C.c_void_p), ("accepted_node", C.c_void_p),
                ("bonus", C.c_void_p), ("row_target", C.c_void_p), ("row_score", C.c_void_p)]


_lib = None


def load(path: str = LIB_PATH):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libspecedge.so not built at {path}; run paper_2505_17052_b200/build.py")
    lib = C.CDLL(path)
    P, I32, U64, SZ = C.c_void_p, C.c_int32, C.c_uint64, C.c_size_t
    sig = {
        "specedge_model_create": [C.POINTER(ModelConfig), U64, I32, C.POINTER(P)],
        "specedge_model_destroy": [P],
        "specedge_kvpool_create": [P, I32, I32, C.POINTER(P)],
        "specedge_kvpool_destroy": [P],
        "specedge_kv_alloc": [P, I32, C.POINTER(I32)],
        "specedge_kv_free": [P, I32],
        "specedge_kv_set_len": [P, P, P, I32, P],
        "specedge_kv_get_len": [P, P, P, I32],
        "specedge_kv_fill_random": [P, I32, I32, U64, C.c_uint32, P],
        "specedge_workspace_size": [P, I32, I32, I32, C.POINTER(SZ)],
        "specedge_prefill": [P, P, I32, P, I32, P, SZ, P],
        "specedge_verify_batch": [P, P, C.POINTER(VerifyIn), C.POINTER(VerifyOut), P, SZ, P],
        "specedge_kv_commit": [P, P, C.POINTER(VerifyIn), C.POINTER(VerifyOut), P, SZ, P],
        "specedge_verify_batch_host": [P, P, C.POINTER(VerifyIn), C.POINTER(VerifyOut), P, SZ, P],
        "specedge_debug_weight_rows": [P, I32, I32, I32, I32, P],
        "specedge_debug_read_kv": [P, I32, I32, I32, I32, I32, P],
        "specedge_debug_read_tree_kv": [P, P, SZ, I32, I32, I32, I32, I32, I32, P],
        "specedge_debug_gemm": [P, P, P, I32, I32, I32, P],
        "specedge_debug_last_logits": [P, P, SZ, I32, I32, P, P],
        "specedge_debug_attention": [P, P, P, P, P, P, I32, I32, I32, I32, I32, P, P, SZ, P],
        "specedge_last_launch_count": [],
        "specedge_graph_stats": [P, P, I32],
        "specedge_tp_fused_mode": [P],
        "specedge_set_kernel_timing": [I32],
        "specedge_kernel_times": [P, P, I32],
        "specedge_tp_unique_id": [P],
        "specedge_model_create_tp": [C.POINTER(ModelConfig), U64, I32, I32, I32, P, C.POINTER(P)],
        "specedge_model_tp_info": [P, P, P, P, P],
        "specedge_tp_fused_enable": [P, I32, P],
        "specedge_calibrate_draft_depth": [C.c_double, C.c_double, C.c_double],
        "specedge_scheduler_create": [C.POINTER(SchedulerConfig), C.POINTER(P)],
        "specedge_scheduler_destroy": [P],
        "specedge_scheduler_admit": [P, C.POINTER(SchedRequest)],
        "specedge_scheduler_plan": [P, P, I32, C.POINTER(I32), C.POINTER(I32)],
        "specedge_scheduler_complete": [P, P, I32, C.c_double],
        "specedge_scheduler_observe": [P, I32, C.c_double],
        "specedge_scheduler_state": [P, P, P, P, P],
        "specedge_draft_tree": [P, P, I32, I32, I32, U64, P, I32, I32, I32, I32, P, SZ, P, P, P, P, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = I32
    _lib = lib
    return lib


def check(status: int, what: str = ""):
    if status != OK:
        raise RuntimeError(f"libspecedge {what} failed with status {status}")
