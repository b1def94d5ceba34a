/*
 * specedge.h — C ABI of libspecedge: B200 (sm_100a) server-side batched verification of
 * edge-drafted token trees, the hot path of SpecEdge (arXiv 2505.17052).
 *
 * What the path computes (citations: P:n = PAPER.md line n, S:n = SPEC.md line n, SURVEY =
 * SURVEY.md section, "amb. Ax" = a reading of an unstated detail, listed in DESIGN.md):
 *   - P:171 (§4.1): "edge GPUs generate candidate tokens and send them to the server, which
 *     verifies them in a single forward pass.  The server returns both the verified tokens
 *     and one additional token", preserving "the exact output distribution of the server
 *     model".
 *   - P:315-316 (§4.3): heterogeneous batches, "custom attention masking for each token
 *     sequence in the batch ... without cross-sequence interference".  (The paper pads KV to
 *     the longest sequence; this library uses a paged, ragged KV cache instead.)
 *   - P:599 (App. A): draft trees of budget 32 pruned by cumulative log-probability.
 *
 * One verify step = tree prep (validate, depth, RoPE position, ancestor bitmask) -> embedding
 * gather -> per layer {RMSNorm, QKV GEMM + RoPE + tree K/V write, tree-masked paged split-KV
 * attention, O-proj + residual, RMSNorm, gate/up GEMM + SwiGLU, down + residual} -> final norm
 * + LM head fused with a vocab-wide argmax (greedy) or Gumbel-max (sampled) reduction, logits
 * never written to HBM -> accept walk + bonus -> KV commit (compaction of the root and the
 * accepted nodes' K/V into the cache).
 *
 * Conventions
 *   - Every function returns a specedge_status: SPECEDGE_OK (0) or a negative API error code.
 *     API errors are detected on the host BEFORE any launch; outputs are then untouched.
 *   - Per-request data errors are written to out->status[r] on the device (positive codes);
 *     an errored request gets accepted_len 0, bonus -1, no commit, and does not affect the
 *     other requests.
 *   - `stream` is a cudaStream_t passed as void*.  Calls are stream-ordered and never
 *     synchronise the host, except the *_host entry points and the setup calls documented as
 *     synchronous.
 *   - "device" pointers are CUDA device memory owned by the caller unless stated otherwise.
 *     The library owns weights, the KV page pool, block tables and the RoPE table.  The
 *     verify workspace is caller-owned (size from specedge_workspace_size).
 *   - Thread safety: one host thread per model / pool at a time.
 */
#ifndef SPECEDGE_H_
#define SPECEDGE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t specedge_status;
typedef struct specedge_model specedge_model;
typedef struct specedge_kvpool specedge_kvpool;

/* ---- API error codes (negative, host-detected) ---- */
#define SPECEDGE_OK 0
#define SPECEDGE_E_INVALID (-1)      /* null pointer, non-positive size, bad mode, bad handle */
#define SPECEDGE_E_CUDA (-2)         /* a CUDA runtime/driver call failed */
#define SPECEDGE_E_OOM (-3)          /* device allocation or KV pages exhausted */
#define SPECEDGE_E_WORKSPACE (-4)    /* workspace too small for this call */
#define SPECEDGE_E_UNSUPPORTED (-5)  /* shape outside what the kernels support */
#define SPECEDGE_E_DEVICE (-6)       /* device is not sm_100 */
#define SPECEDGE_E_PROTOCOL (-7)     /* scheduler: a session already has an outstanding request */

/* ---- per-request status codes (device-written, out->status[r]) ---- */
#define SPECEDGE_REQ_OK 0
#define SPECEDGE_REQ_E_TREE 1         /* parent[i] not in {-1} U [0, i) */
#define SPECEDGE_REQ_E_TREE_SIZE 2    /* N > 64 nodes                            (amb. A5) */
#define SPECEDGE_REQ_E_TOKEN 3        /* root or draft token outside [0, V)              */
#define SPECEDGE_REQ_E_DUP_SIBLING 4  /* two children of one parent share a token */
#define SPECEDGE_REQ_E_CONTEXT 5      /* context_len != cached + 1, or > max_context_len, or a
                                         tree position cached + depth >= max_position
                                         ("context-length mismatch -> protocol error") */
#define SPECEDGE_REQ_E_KV_CAPACITY 6  /* cached + deepest path + 1 exceeds the handle's capacity */
#define SPECEDGE_REQ_E_HANDLE 7       /* KV handle not allocated */
#define SPECEDGE_REQ_E_UNSUPPORTED 8  /* SAMPLE_PQ_DENSE: the draft is not a chain */
/* validation order (first failing check wins): HANDLE, TREE_SIZE, TREE, TOKEN, DUP_SIBLING,
   CONTEXT, KV_CAPACITY — identical to oracle/verify.py:validate for the shared codes. */

/* ---- verification modes (SURVEY amb. A7-A9) ---- */
#define SPECEDGE_GREEDY 0       /* y = argmax_v logit, ties -> lowest id */
#define SPECEDGE_SAMPLE_TREE 1  /* y = argmax_v (logit/T + Gumbel(seed, round, session, slot, v)) */
/* NEXT-F2: speculative sampling of a chain whose tokens the edge SAMPLED from its
 * draft distributions q, shipped dense in verify_in.draft_q (App. B, P:766-770:
 * Leviathan et al.).  Node i is accepted iff u(slot i) < p_i(x_i) / q_i(x_i),
 * p_i = softmax(l / T) at slot i; the first rejection's bonus is drawn from norm(max(0, p - q))
 * by Gumbel-max over log(max(0, p - q)), after full acceptance from p at the last slot.
 * u(slot) = ((w >> 8) | 1) 2^-24, w = Philox4x32-10 word 0 of counter (slot, 'ACPT',
 * lo32(session), hi32(session)), key (lo32(seed) ^ round, hi32(seed)).  Requires T >= 1e-6,
 * draft_q != NULL and tp_size == 1 (else E_INVALID / E_UNSUPPORTED); a request whose tree is not
 * a chain gets status REQ_E_UNSUPPORTED.  Cost: two LM-head passes (log-sum-exp, then residual). */
#define SPECEDGE_SAMPLE_PQ_DENSE 2

#define SPECEDGE_MAX_NODES 64
#define SPECEDGE_PAGE_TOKENS 64

/* Decoder shape (Llama/Qwen3 family, SURVEY amb. A13-A16; no biases, untied LM head).
 * Supported: head_dim in {16, 32, 64, 128}; d, n_heads*head_dim, ffn multiples of 64;
 * n_heads % n_kv == 0. */
typedef struct {
  int32_t n_layers, d, n_heads, n_kv, head_dim, ffn, vocab;
  float eps;            /* RMSNorm epsilon */
  double rope_theta;    /* RoPE base (rotate-half convention, amb. A14) */
  int32_t max_position; /* RoPE table length; positions must be < max_position */
} specedge_model_config;

/* Create a model on `device` with synthetic bf16 weights that are a pure function of
 * `weight_seed` (Philox4x32-10, generated on the device; bit-identical to the
 * oracle's generator).  Synchronous.  *out receives an owned handle. */
specedge_status specedge_model_create(const specedge_model_config* cfg, uint64_t weight_seed,
                                      int32_t device, specedge_model** out);
specedge_status specedge_model_destroy(specedge_model* model);

/* ---- tensor parallelism (SURVEY §8(a) a12, §8(e) "Tensor parallel TP = 8"; cfg4) ----
 * One process per GPU; every rank creates its shard with the same cfg / weight_seed and the
 * same 128-byte NCCL unique id (from specedge_tp_unique_id on one rank, broadcast by the caller).
 * Rank k holds: q heads [k*H/tp, (k+1)*H/tp) and kv heads [k*KV/tp, ...) (head-parallel attention;
 * the KV pool of this model stores only those kv heads), gate/up rows [k*F/tp, ...) (column
 * parallel), the matching input columns of Wo and Wd (row parallel; their fp32 [R, d] outputs
 * are summed over ranks by an NCCL all-reduce on the verify stream: C1 after O, C2 after down),
 * the LM-head rows [v0, v0+vn) with vn = ceil(V/tp) (vocab parallel; the per-row (score, id)
 * winners are all-gathered and reduced, ties -> lowest id: C3).  Embedding, norms, walk and
 * commit are replicated.  Every shard is bit-identical to the corresponding slice of the
 * tp_size == 1 model.  Requires n_heads, n_kv divisible by tp_size and ffn by 64*tp_size, else
 * E_UNSUPPORTED; E_UNSUPPORTED also when libnccl.so.2 cannot be loaded.  All ranks must call
 * every verify / prefill with identical inputs (collectives are issued in program order).
 * Synchronous (NCCL communicator creation blocks until all ranks joined). */
specedge_status specedge_tp_unique_id(uint8_t* nccl_id /* [128] host */);
specedge_status specedge_model_create_tp(const specedge_model_config* cfg, uint64_t weight_seed,
                                         int32_t device, int32_t tp_rank, int32_t tp_size,
                                         const uint8_t* nccl_id /* [128] host; see below */,
                                         specedge_model** out);
/* nccl_id == NULL with tp_size > 1 creates a communicator-less shard: weights, KV pool and the
 * debug introspection work (one process can compare every shard with the tp_size == 1 model on
 * one GPU), verify / prefill return E_UNSUPPORTED. */
/* This rank's position and LM-head vocab shard [vocab0, vocab0 + vocab_n); NULL outputs skipped. */
specedge_status specedge_model_tp_info(const specedge_model* model, int32_t* tp_rank,
                                       int32_t* tp_size, int32_t* vocab0, int32_t* vocab_n);
/* NEXT-F4: fuse the reduce-scatter of the row-parallel O / down GEMMs' fp32 [R, d]
 * updates (C1, C2 of specedge_model_create_tp) into the kernels over NVLink peer memory.
 * Collective: every rank calls it once, with the same max_rows, before verifying.  Allocates this
 * rank's exchange buffer (max(max_rows, 2 x tp_size x ceil(max_rows / tp_size)) x d fp32) and flag
 * words, exchanges CUDA IPC handles over the model's NCCL communicator and maps every peer's
 * buffer.  Afterwards a verify of R <= max_rows rows runs C1/C2 without NCCL: by default the GEMM
 * epilogue stages each 32-row chunk in shared memory and bulk-copies every row to the receive slot
 * of the rank that owns it (environment SPECEDGE_TP_F4=pull instead writes locally and lets the
 * owner's RMSNorm load its rows from every rank); an epoch flag is released on every peer after
 * the GEMM and the owner's RMSNorm, after acquiring the flags, sums the tp slots in rank order
 * (deterministic).  Larger R use the NCCL path.
 * E_INVALID: tp_size < 2 or > 4, max_rows <= 0, or already enabled with a smaller max_rows;
 * E_CUDA: allocation / IPC / NCCL failure (the model stays on the NCCL path).  Synchronous;
 * `stream` carries the handle all-gather. */
specedge_status specedge_tp_fused_enable(specedge_model* model, int32_t max_rows, void* stream);
/* The reduce-scatter path in effect: 0 NCCL (fused path off), 1 push (epilogue bulk copies into the
 * owners' receive slots), 2 pull (SPECEDGE_TP_F4=pull: the owner's RMSNorm loads every rank's rows),
 * 3 NVLS (SPECEDGE_TP_F4=nvls: every rank's partial lives in its own buffer bound to one CUDA
 * multicast object; the owner's RMSNorm loads the rank sum with multimem.ld_reduce, reduced in
 * the NVSwitch).  NVLS falls back to push, on every rank, when the multicast object cannot be set
 * up (no multicast support, file-descriptor exchange refused).  Host only. */
int32_t specedge_tp_fused_mode(const specedge_model* model);

/* KV page pool of `num_pages` pages x 64 tokens x all layers (fp16 K and V), zero-initialised,
 * with room for `max_handles` sessions.  Synchronous. */
specedge_status specedge_kvpool_create(specedge_model* model, int32_t num_pages,
                                       int32_t max_handles, specedge_kvpool** out);
specedge_status specedge_kvpool_destroy(specedge_kvpool* pool);
/* Reserve pages for a session able to hold `capacity_tokens` cached tokens; returns the handle
 * (>= 0) in *out_handle with cached length 0.  E_OOM if pages or handles are exhausted;
 * E_INVALID if capacity_tokens <= 0 or > the model's max_position (RoPE table length).
 * Synchronous (host allocator + one small H2D copy). */
specedge_status specedge_kv_alloc(specedge_kvpool* pool, int32_t capacity_tokens,
                                  int32_t* out_handle);
specedge_status specedge_kv_free(specedge_kvpool* pool, int32_t handle);
/* Set the cached length of n sessions (host arrays), stream-ordered (used to rewind a session
 * between benchmark steps).  Lengths must be <= capacity.  The values travel as kernel
 * parameters: the host arrays may be reused on return and the call can be captured in a CUDA
 * graph. */
specedge_status specedge_kv_set_len(specedge_kvpool* pool, const int32_t* handles,
                                    const int32_t* lens, int32_t n, void* stream);
/* Read the cached lengths of n sessions into host array `lens` (synchronous). */
specedge_status specedge_kv_get_len(specedge_kvpool* pool, const int32_t* handles, int32_t* lens,
                                    int32_t n);
/* Fill positions [0, n_tokens) of a session with synthetic K/V (element =
 * fp16(int24 * 2^-23) from Philox keyed (seed, position, layer*2+kv, stream_id ^ 'KVFI')) and
 * set its cached length to n_tokens.  Performance runs only; parity runs prefill for real. */
specedge_status specedge_kv_fill_random(specedge_kvpool* pool, int32_t handle, int32_t n_tokens,
                                        uint64_t seed, uint32_t stream_id, void* stream);

/* Bytes of workspace a verify / prefill call needs for up to max_requests requests,
 * max_rows = sum of (nodes + 1) rows, and contexts up to max_context_len tokens. */
specedge_status specedge_workspace_size(const specedge_model* model, int32_t max_requests,
                                        int32_t max_rows, int32_t max_context_len,
                                        size_t* bytes);

/* Prefill (outside the measured path): run the decoder over host tokens[0..n-2] of a
 * session and append their K/V to its cache (chunked causal chain verification on the same
 * kernels; chunks of up to 65 rows, fewer if the workspace is smaller).  tokens[n-1] becomes the
 * next root.  Synchronous (checks each chunk's status); E_INVALID on a bad token or handle. */
specedge_status specedge_prefill(specedge_model* model, specedge_kvpool* pool, int32_t handle,
                                 const int32_t* tokens_host, int32_t n, void* workspace,
                                 size_t ws_bytes, void* stream);

/* ---- the hot path ---- */
typedef struct {
  /* host scalars */
  int32_t num_requests;     /* B >= 1 */
  int32_t total_nodes;      /* sum_r N_r (root excluded, amb. A1); rows R = total_nodes + B */
  int32_t max_nodes;        /* >= max_r N_r, <= 64 */
  int32_t max_context_len;  /* >= max_r context_len[r] (grid sizing; checked per request) */
  int32_t mode;             /* SPECEDGE_GREEDY | SPECEDGE_SAMPLE_TREE */
  float temperature;        /* used iff mode == SAMPLE_TREE; T < 1e-6 => GREEDY */
  uint64_t seed;            /* sampling seed (amb. A9) */
  int32_t auto_commit;      /* 1: also commit accepted K/V (== calling specedge_kv_commit) */
  /* device arrays (caller-owned, valid until the stream passes this call) */
  const int32_t* kv;             /* [B] KV handle per request */
  const int32_t* context_len;    /* [B] committed tokens C_r = cached + 1 (amb. A2) */
  const int32_t* root_token;     /* [B] last committed token (previous bonus) */
  const uint64_t* session_id;    /* [B] RNG key part */
  const uint32_t* round;         /* [B] RNG key part: per-session verify counter */
  const int32_t* node_offset;    /* [B+1] CSR offsets into the node arrays */
  const int32_t* parent;         /* [total_nodes] -1 = child of root, else local index < i */
  const int32_t* token;          /* [total_nodes] draft tokens */
  const float* draft_logprob;    /* [total_nodes] log q, nullable; unused by GREEDY and
                                    SAMPLE_TREE (SURVEY Lemma, amb. A23) */
  const float* draft_q;          /* [total_nodes][V] fp32 draft distributions, row i = the q
                                    node i was sampled from; SAMPLE_PQ_DENSE only, else NULL */
} specedge_verify_in;

typedef struct {                 /* device arrays, caller-allocated */
  int32_t* status;               /* [B] per-request status (SPECEDGE_REQ_*) */
  int32_t* accepted_len;         /* [B] a_r: accepted draft nodes (tokens/verify = a_r + 1) */
  int32_t* accepted_token;       /* [total_nodes] CSR by node_offset, first a_r valid */
  int32_t* accepted_node;        /* [total_nodes] node indices of the accepted root path */
  int32_t* bonus;                /* [B] the one additional token; -1 on error */
  int32_t* row_target;           /* [R] nullable: target token y per slot (slot 0 = root) */
  float* row_score;              /* [R] nullable: top-1 score (max logit, or max Gumbel score) */
} specedge_verify_out;

/* Verify a batch.  Row r's slots occupy rows node_offset[r] + r ... node_offset[r+1] + r
 * (slot 0 = root, slot i+1 = node i).  Errors: E_INVALID (null/mismatched arguments,
 * max_nodes > 64, bad mode), E_WORKSPACE, E_UNSUPPORTED, E_CUDA. */
specedge_status specedge_verify_batch(specedge_model* model, specedge_kvpool* pool,
                                      const specedge_verify_in* in, specedge_verify_out* out,
                                      void* workspace, size_t ws_bytes, void* stream);

/* Commit the K/V of the root and the accepted nodes of a previous verify_batch (same `in`,
 * `out`, same workspace, no other verify on that workspace in between).  Applies at most once:
 * a request whose cached length already moved is skipped and gets status E_CONTEXT. */
specedge_status specedge_kv_commit(specedge_model* model, specedge_kvpool* pool,
                                   const specedge_verify_in* in, specedge_verify_out* out,
                                   void* workspace, size_t ws_bytes, void* stream);

/* End-to-end entry point with HOST buffers (same fields; every pointer in `in`/`out` is host
 * memory, pinned for best results).  Copies the inputs into the workspace, verifies, copies
 * the outputs back and synchronises `stream` before returning.  SAMPLE_PQ_DENSE (dense q rows)
 * is device-entry only here: E_UNSUPPORTED. */
specedge_status specedge_verify_batch_host(specedge_model* model, specedge_kvpool* pool,
                                           const specedge_verify_in* in_host,
                                           specedge_verify_out* out_host, void* workspace,
                                           size_t ws_bytes, void* stream);

/* ---- test introspection (used by tests/ only; never on the verify path) ---- */
/* Logical weight rows back to the host as bf16 bits: tensor ids as in oracle/model.py
 * (1 embed, 2 wq, 3 wk, 4 wv, 5 wo, 6 wg, 7 wu, 8 wd, 9 lm_head, 10 g_attn, 11 g_mlp,
 * 12 g_final).  Of a tensor-parallel shard: its local rows and columns (row 0 of lm_head = vocab
 * id vocab0).  Synchronous. */
specedge_status specedge_debug_weight_rows(specedge_model* model, int32_t tensor, int32_t layer,
                                           int32_t row0, int32_t nrows, uint16_t* dst_host);
/* Cached K or V (kv_sel 0/1) of positions [pos0, pos0+n) of a session, layer `layer`, as fp16
 * bits [n][n_kv][head_dim] into host memory (the KV cache is fp16).  Synchronous. */
specedge_status specedge_debug_read_kv(specedge_kvpool* pool, int32_t handle, int32_t layer,
                                       int32_t kv_sel, int32_t pos0, int32_t n,
                                       uint16_t* dst_host);
/* Tree K/V scratch of the last verify with this workspace and batch size (num_requests B,
 * rows R = total_nodes + B): K or V (kv_sel 0/1) of rows [row0, row0+n) of `layer`, as fp16 bits
 * [n][n_kv][head_dim] into host memory.  Row node_offset[r] + r is request r's root slot, the next
 * N_r rows its nodes (the rows a commit copies into the pages).  Synchronous. */
specedge_status specedge_debug_read_tree_kv(specedge_model* model, const void* workspace,
                                            size_t ws_bytes, int32_t num_requests, int32_t R,
                                            int32_t layer, int32_t kv_sel, int32_t row0,
                                            int32_t n, uint16_t* dst_host);
/* Run the tcgen05 GEMM alone: out[r][m] = sum_k X[r][k] * W[m][k] (bf16 in, fp32 out), all
 * device pointers, row-major.  M, K multiples of 64 (M tile zero-padded), R >= 1. */
specedge_status specedge_debug_gemm(const uint16_t* W, const uint16_t* X, float* out, int32_t M,
                                    int32_t R, int32_t K, void* stream);
/* Run the LM-head GEMM (same tcgen05 kernel, fp32-store epilogue) on the final-norm hidden
 * states left in the workspace by the last verify of (num_requests, R): writes fp32 logits
 * [R][vocab_n] (this rank's vocab shard, all of V when tp_size == 1) to logits_dev.  Test-only; the verify path itself never materialises logits. */
specedge_status specedge_debug_last_logits(specedge_model* model, void* workspace,
                                           size_t ws_bytes, int32_t num_requests, int32_t R,
                                           float* logits_dev, void* stream);
/* Tree-masked attention kernel alone on caller data (all device): q [S][G][hd] fp16 for one
 * request and one kv head, prefix k/v [L][hd] fp16, tree k/v [S][hd] fp16, anc [S-1] uint64
 * (ancestor-or-self masks over nodes); writes o [S][G][hd] fp32 (normalised). */
specedge_status specedge_debug_attention(const uint16_t* q, const uint16_t* k_prefix,
                                         const uint16_t* v_prefix, const uint16_t* k_tree,
                                         const uint16_t* v_tree, const uint64_t* anc, int32_t S,
                                         int32_t G, int32_t head_dim, int32_t L,
                                         int32_t n_splits, float* o, void* workspace,
                                         size_t ws_bytes, void* stream);

/* CUDA-graph cache of whole verify steps: out3 = {replays of a cached graph, captures (a
 * signature's second use), plain launches (a signature's first use)} since the last reset.  A
 * signature is (num_requests, total_nodes, max_nodes, max_context_len, mode, temperature, seed,
 * auto_commit, buffer addresses): a serving loop that keeps its buffers and passes a constant
 * max_context_len bound reuses one graph per (batch size, node count).  Host only. */
specedge_status specedge_graph_stats(const specedge_model* model, int64_t* out3, int32_t reset);

/* Number of kernels the last verify_batch call launched (host counter, for the benchmark's
 * gpu_launches field). */
int32_t specedge_last_launch_count(void);

/* ---- per-kernel timing (benchmark instrumentation) ----
 * enable: 0 off, -1 every kernel kind, > 0 bitmask of kinds (bit k = kind k).  When enabled,
 * verify_batch records a CUDA event pair on `stream` around every launch of a selected kind
 * (stream-ordered, no host sync; each pair costs a few microseconds of stream time).  specedge_kernel_times synchronises on the recorded
 * events, adds their durations to per-kind totals and clears the pending list; out_ms[k] and
 * out_count[k] (arrays of SPECEDGE_KERNEL_KINDS) receive the totals since the last reset.
 * Kinds: 0 prep, 1 embed, 2 rmsnorm, 3 gemm_qkv, 4 attention, 5 attn_combine, 6 gemm_o,
 * 7 gemm_gateup, 8 gemm_down, 9 gemm_lmhead, 10 lm_reduce, 11 walk, 12 commit, 13 qkv_rope. */
#define SPECEDGE_KERNEL_KINDS 14
specedge_status specedge_set_kernel_timing(int32_t enable);
specedge_status specedge_kernel_times(float* out_ms, int32_t* out_count, int32_t reset);

/* ---- NEXT-F1: pipeline-aware verification scheduler (host only) ----
 * PAPER.md §4.3: the server interleaves verification of many sessions and "dynamically
 * calibrates ... draft depth" so that "server verification time ~= edge drafting time + network
 * round-trip time"; worked depths in §5.2 (94.2 ms verify, 11 ms per draft pass ->
 * depth 7 / 5 / 4 at RTT 15 / 40 / 50 ms).  Interface after SPEC.md S:311-383.  The scheduler is a
 * single-threaded decision point in front of specedge_verify_batch; it never touches the GPU.
 * Readings (DESIGN.md §4 R-sched): depth = max(1, round-half-away((verify - rtt) / draft_pass));
 * estimates are exponentially weighted means (weight w, S:322 default 0.2) whose first observation
 * initialises them unless a positive prior is configured; FIFO by (arrival, admission order);
 * work-conserving plans of the oldest min(capacity, queued) requests. */
#define SPECEDGE_TIMING_VERIFY 0       /* server verify-step time (ms) */
#define SPECEDGE_TIMING_DRAFT_PASS 1   /* one edge draft forward pass (ms) */
#define SPECEDGE_TIMING_RTT 2          /* network round trip (ms) */

typedef struct specedge_scheduler specedge_scheduler;
typedef struct {
  int32_t capacity;           /* max requests per verify batch, >= 1 */
  double ewma_weight;         /* in (0, 1] */
  int32_t fixed_depth;        /* > 0: always this depth; 0: calibrate */
  double init_verify_ms;      /* priors (<= 0: none, the first observation initialises) */
  double init_draft_pass_ms;
  double init_rtt_ms;
} specedge_scheduler_config;

typedef struct {              /* one pending verify request (host values, copied) */
  uint64_t session_id;
  int32_t kv_handle;
  int32_t length;             /* committed context + draft nodes (reported as padded_len) */
  double arrival_ms;          /* caller's clock */
} specedge_sched_request;

/* Pure depth rule; returns >= 1 (draft_pass_ms <= 0 or non-finite input -> 1). */
int32_t specedge_calibrate_draft_depth(double verify_ms, double draft_pass_ms, double rtt_ms);
specedge_status specedge_scheduler_create(const specedge_scheduler_config* cfg,
                                          specedge_scheduler** out);
specedge_status specedge_scheduler_destroy(specedge_scheduler* sched);
/* Enqueue; E_PROTOCOL if the session is already queued or in service. */
specedge_status specedge_scheduler_admit(specedge_scheduler* sched, const specedge_sched_request* req);
/* Dequeue the oldest min(capacity, max_members, queued) requests into members[] (in order), set
 * *n_members (0 when the queue is empty) and *padded_len = max member length (nullable).  The
 * members stay outstanding until specedge_scheduler_complete. */
specedge_status specedge_scheduler_plan(specedge_scheduler* sched, specedge_sched_request* members,
                                        int32_t max_members, int32_t* n_members, int32_t* padded_len);
/* A batch finished after verify_ms: its sessions may be admitted again; updates the verify estimate. */
specedge_status specedge_scheduler_complete(specedge_scheduler* sched, const uint64_t* sessions,
                                            int32_t n, double verify_ms);
/* Feed a timing measurement (kind = SPECEDGE_TIMING_*). */
specedge_status specedge_scheduler_observe(specedge_scheduler* sched, int32_t kind, double ms);
/* Current draft depth, queue size, outstanding sessions and the three estimates (-1 = none yet);
 * every output nullable. */
specedge_status specedge_scheduler_state(const specedge_scheduler* sched, int32_t* depth,
                                         int32_t* queued, int32_t* outstanding, double* estimates3);

/* ---- NEXT-F3: draft-tree builder (edge side) ----
 * PAPER.md App. A: draft passes propose parallel candidates "pruned based on cumulative log
 * probabilities so that the total number of tokens remains within the tree budget".  Runs `depth`
 * passes of this model (the draft model) over the session `handle` (context_len = cached + 1,
 * root_token = its last committed token): every frontier node proposes its top-`branching` tokens
 * (ties: smaller id, log-softmax at T = 1), proposals are pooled with the kept nodes and the first
 * `budget` in (-cum logprob, depth, token, insertion) order are kept (ancestor-closed), in
 * insertion order (DESIGN.md R-draft).  Each pass is the verify path up to the
 * final norm on a one-request tree, the LM head with an fp32 store epilogue and a top-b kernel;
 * pruning is host code.  Outputs (host arrays of >= budget entries): parent (-1 = root child, else
 * a smaller index), token, logprob; *n_out = node count.  Synchronous.  budget <= 64, branching <= 8,
 * tp_size == 1; the workspace must fit (1 request, head_len + budget + 1 rows).  Does not commit.
 * Proactive expansion (§4.2: the edge "continues drafting additional tokens"
 * from the best path's leaf while the verify is in flight): head_tokens[head_len] (host, nullable
 * when head_len = 0) is that path below the root; the subtree grows under its last token and the
 * outputs describe the subtree only (parent -1 = child of the head; logprobs of the subtree nodes). */
specedge_status specedge_draft_tree(specedge_model* model, specedge_kvpool* pool, int32_t handle,
                                    int32_t context_len, int32_t root_token, uint64_t session_id,
                                    const int32_t* head_tokens, int32_t head_len, int32_t budget,
                                    int32_t depth, int32_t branching, void* workspace, size_t ws_bytes,
                                    void* stream, int32_t* parent_out, int32_t* token_out,
                                    float* logprob_out, int32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* SPECEDGE_H_ */
