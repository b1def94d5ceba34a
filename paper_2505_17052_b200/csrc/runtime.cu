// libspecedge runtime: model / KV pool / workspace management and the C ABI (include/specedge.h).
// The verify step is a fixed stream-ordered sequence of sm_100a kernels; the host only checks
// arguments, sizes the launches and encodes TMA descriptors.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <string>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

using namespace se;

namespace {
std::mutex g_carve_mu;
std::set<std::pair<const void*, int>> g_carve_seen;
}  // namespace
int se::carveout_mode() {
  static const int m = getenv("SPECEDGE_CARVEOUT") ? atoi(getenv("SPECEDGE_CARVEOUT")) : 1;
  return m;
}
bool se::carveout_first(const void* kern) {
  if (carveout_mode() == 0) return false;
  std::lock_guard<std::mutex> lk(g_carve_mu);
  return g_carve_seen.insert({kern, current_device()}).second;
}
void se::carveout_skip(const void* kern) {
  std::lock_guard<std::mutex> lk(g_carve_mu);
  g_carve_seen.insert({kern, current_device()});
}

// Programmatic dependent launch: on by default (SPECEDGE_PDL=0 disables).  Every kernel calls
// pdl_begin() (trigger, then griddepcontrol.wait) before its first global access, so the next
// kernel's CTAs are resident and set up when the previous one drains.  Measured on cfg2 with every
// kernel at the max-shared carveout: +1.2 % device / +3 % e2e tok/s (3 alternating pairs, one box;
// round 1, with mixed carveouts: no change); the full GPU suite passes with it.
bool se::pdl_enabled() {
  static const bool on = !(getenv("SPECEDGE_PDL") && getenv("SPECEDGE_PDL")[0] == '0');
  return on;
}

namespace {

// Tree attention work split on the tcgen05 path: the persistent, evenly split grid
// (attention_tc.cu, per_req = 2) for long contexts (>= kBalancedPages pages of 64 keys), else
// one CTA per (request, kv head, chunk).  Measured (profiles/README.md): cfg5 (12k-20k
// contexts) gains, cfg2 (1k) loses (every pass of its replicated tail tile drains the ring).
// SPECEDGE_ATTN_BALANCED=0/1 forces either.
bool attn_balanced(int max_pages) {
  static const int force = getenv("SPECEDGE_ATTN_BALANCED") ? atoi(getenv("SPECEDGE_ATTN_BALANCED")) : -1;
  static const int min_pages = getenv("SPECEDGE_ATTN_BAL_PAGES") ? atoi(getenv("SPECEDGE_ATTN_BAL_PAGES")) : 64;
  return force >= 0 ? force == 1 : max_pages >= min_pages;
}
int num_sms() { return device_sms(); }
// a9: hi-only LM head + exact candidate rescoring (default), or the hi/lo operand pair through the
// MMA for every vocab id (SPECEDGE_LM_PAIR=1)
bool lm_hi_only() {
  static const bool pair = getenv("SPECEDGE_LM_PAIR") && getenv("SPECEDGE_LM_PAIR")[0] == '1';
  return !pair;
}

thread_local int g_last_launches = 0;

// K-split cap per fp32 GEMM kind (consumers sum the partials: RoPE after QKV, RMSNorm after O /
// down).  Env SPECEDGE_SPLITS_QKV / _O / _DOWN override (A/B); defaults from cfg2 measurements.
int kind_splits(int kind);

// ---- optional per-kernel event timing (bench instrumentation) ----
enum Kind { K_PREP, K_EMBED, K_RMSNORM, K_QKV, K_ATTN, K_COMBINE, K_O, K_GU, K_DOWN, K_LM, K_LMRED, K_WALK, K_COMMIT,
            K_ROPE, K_NKINDS };
int kind_splits(int kind) {
  auto env = [](const char* n, int d) { return getenv(n) ? std::max(1, atoi(getenv(n))) : d; };
  static const int qkv = env("SPECEDGE_SPLITS_QKV", 4), o = env("SPECEDGE_SPLITS_O", 4), down = env("SPECEDGE_SPLITS_DOWN", 4);
  return kind == K_QKV ? qkv : (kind == K_O ? o : (kind == K_DOWN ? down : 4));
}
struct Timing {
  bool on = false;
  uint32_t mask = 0;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<int, size_t>> pending;   // (kind, index of start event)
  double ms[K_NKINDS] = {};
  int count[K_NKINDS] = {};
} g_timing;

cudaEvent_t timing_event() {
  if (g_timing.used == g_timing.pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_timing.pool.push_back(e);
  }
  return g_timing.pool[g_timing.used++];
}

// RAII: records a start event on construction and an end event on destruction (if enabled)
struct KTimer {
  int kind;
  cudaStream_t st;
  size_t idx = 0;
  bool active = false;
  KTimer(int k, cudaStream_t s) : kind(k), st(s) {
    active = g_timing.on && ((g_timing.mask >> k) & 1u);
    if (!active) return;
    idx = g_timing.used;
    record(timing_event());
  }
  ~KTimer() {
    if (!active) return;
    record(timing_event());
    g_timing.pending.push_back({kind, idx});
  }
  // under stream capture an event must be an external record node to be timed on each replay
  void record(cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
  }
};

// SPECEDGE_DEBUG=1: name the failing call on stderr
thread_local int g_dbg_layer = -1;
bool ck_debug() {
  static const bool on = getenv("SPECEDGE_DEBUG") && getenv("SPECEDGE_DEBUG")[0] == '1';
  return on;
}
#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t _e = (x);                                                                         \
    if (_e != cudaSuccess) {                                                                      \
      if (ck_debug()) fprintf(stderr, "libspecedge: %s:%d (layer %d) %s -> %s\n", __FILE__, __LINE__, \
                              g_dbg_layer, #x, cudaGetErrorString(_e));                           \
      return SPECEDGE_E_CUDA;                                                                     \
    }                                                                                             \
  } while (0)

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
  size_t req_L, req_h, req_row0, req_S, row_tok, row_pos, row_req, row_slot, row_anc;
  size_t X, Y, Hn, Hf, Q, O, M, tree_kv, opart, mpart, lpart, attn_nch, attn_cnt, part_val, part_idx, part_val2, part_idx2, part_val3,
      tile_cnt, y, score, tp_gather;
  size_t part_m, part_s, lse, row_qnode, pchild, resid_y, resid_s;   // SAMPLE_PQ_DENSE
  size_t draft_logits;                                                // [R][V] fp32 logits of a draft pass (NEXT-F3 only)
  size_t stage_in, stage_out, total, tile_cnt_bytes;
  int B, R, n_splits_max;
};

constexpr int kMaxSplits = 8;
constexpr int kGemmSplits = 4;

WsLayout ws_layout(const specedge_model_config& c, int B, int R) {
  WsLayout w{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = al256(o + bytes);
    return at;
  };
  const size_t H = c.n_heads, hd = c.head_dim, KV = c.n_kv;
  w.req_L = take(4 * B);
  w.req_h = take(4 * B);
  w.req_row0 = take(4 * B);
  w.req_S = take(4 * B);
  w.row_tok = take(4 * R);
  w.row_pos = take(4 * R);
  w.row_req = take(4 * R);
  w.row_slot = take(4 * R);
  w.row_anc = take(8 * R);
  // row buffers carry kMaxTp spare rows: under tensor parallelism the residual stream is
  // row-sharded in equal chunks of ceil(R / tp) rows (reduce-scatter / all-gather)
  const size_t Rp = (size_t)R + kMaxTp;
  w.X = take(4 * Rp * c.d);   // fp32 residual stream
  // fp32 K-split partials of the QKV / O / down GEMMs: [kGemmSplits][Rp][max(qkv, d)]
  w.Y = take(4 * (size_t)kGemmSplits * Rp * std::max((size_t)(H + 2 * KV) * hd, (size_t)c.d));
  w.Hn = take(2 * Rp * c.d);
  w.Hf = take(2 * 2 * Rp * c.d);   // final-norm output as hi/lo bf16 row pairs
  w.Q = take(2 * (size_t)R * H * hd);
  w.O = take(2 * (size_t)R * H * hd);
  w.M = take(2 * (size_t)R * c.ffn);
  w.tree_kv = take(2 * (size_t)c.n_layers * 2 * KV * R * hd);
  w.opart = take(4 * (size_t)kMaxSplits * R * H * hd);
  w.mpart = take(4 * (size_t)kMaxSplits * R * H);
  w.lpart = take(4 * (size_t)kMaxSplits * R * H);
  w.attn_nch = take(4 * (size_t)B * KV);   // balanced attention: chunks per (request, kv head)
  w.attn_cnt = take(4 * (size_t)B * KV);   // balanced attention: finished-chunk counters
  const size_t vt = (c.vocab + 127) / 128;
  w.part_val = take(4 * (size_t)R * vt);
  w.part_idx = take(4 * (size_t)R * vt);
  w.part_val2 = take(4 * (size_t)R * vt);
  // fused residual add: one counter per (256-feature tile, row tile, multicast slot, CTA half)
  // + 2048 counters for the SwiGLU GEMM's last-wave K-parts (< 256 clusters x <= 4 pairs x 2 halves)
  w.tile_cnt_bytes = 4 * (size_t)((c.d + 255) / 256) * ((R + 15) / 16 + 1) * 4 * 2 + 4 * 2048;
  w.tile_cnt = take(w.tile_cnt_bytes);
  w.part_idx2 = take(4 * (size_t)R * vt);
  w.part_val3 = take(4 * (size_t)R * vt);
  w.y = take(4 * R);
  w.score = take(4 * R);
  w.tp_gather = take(8 * (size_t)(kMaxTp + 1) * R);   // TP C3: [tp][R](score, id) + own staging
  w.part_m = take(4 * (size_t)R * vt);
  w.part_s = take(4 * (size_t)R * vt);
  w.lse = take(4 * R);
  w.row_qnode = take(4 * R);
  w.pchild = take(4 * R);
  w.resid_y = take(4 * R);
  w.resid_s = take(4 * R);
  w.draft_logits = take(4 * (size_t)R * c.vocab);
  // staging for the host-buffer entry point: inputs then outputs
  w.stage_in = take((size_t)B * (4 + 4 + 4 + 8 + 4) + 4 * (B + 1) + (size_t)R * 12 + 64);
  w.stage_out = take((size_t)B * 12 + (size_t)R * 8 + (size_t)R * 8 + 64);
  w.total = o;
  w.B = B;
  w.R = R;
  w.n_splits_max = kMaxSplits;
  return w;
}

bool check_cfg(const specedge_model_config& c) {
  if (c.n_layers <= 0 || c.d <= 0 || c.n_heads <= 0 || c.n_kv <= 0 || c.ffn <= 0 || c.vocab <= 0) return false;
  if (c.n_heads % c.n_kv) return false;
  if (!(c.head_dim == 16 || c.head_dim == 32 || c.head_dim == 64 || c.head_dim == 128)) return false;
  if (c.d % 64 || (c.n_heads * c.head_dim) % 64 || c.ffn % 64 || c.d > 16384) return false;
  if (c.max_position <= 0) return false;
  return true;
}

template <typename T>
T* dalloc(specedge_model* m, size_t n) {
  void* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return nullptr;
  m->allocs.push_back(p);
  return reinterpret_cast<T*>(p);
}

struct DevIn {
  const int32_t *kv, *context_len, *root_token, *node_offset, *parent, *token;
  const uint64_t* session_id;
  const uint32_t* round;
};

struct DevOut {
  int32_t *status, *accepted_len, *accepted_token, *accepted_node, *bonus, *row_target;
  float* row_score;
};

// hidden_only (NEXT-F3 draft passes): stop after the final RMSNorm (hi/lo rows in ws Hf); no LM
// head, walk or commit
specedge_status run_verify(specedge_model* m, specedge_kvpool* pool, const specedge_verify_in* in, DevIn di,
                           DevOut dout, uint8_t* ws_base, size_t ws_bytes, cudaStream_t st, bool prefill,
                           bool do_commit, bool hidden_only = false) {
  const specedge_model_config& c = m->cfg;
  if (m->tp_size > 1 && !m->nccl) return SPECEDGE_E_UNSUPPORTED;   // a communicator-less shard
  const int B = in->num_requests, T = in->total_nodes, R = T + B;
  const WsLayout w = ws_layout(c, B, R);
  if (!ws_base || ws_bytes < w.total) return SPECEDGE_E_WORKSPACE;
  uint8_t* ws = ws_base;
  auto P = [&](size_t off) { return ws + off; };
  int launches = 0;
  const int R_cap = R;

  PrepArgs pa{};
  pa.B = B;
  pa.V = c.vocab;
  pa.max_nodes = in->max_nodes;
  pa.max_context_len = in->max_context_len;
  pa.max_handles = pool->max_handles;
  pa.force_chain = prefill ? 1 : 0;
  pa.max_position = c.max_position;   // RoPE table rows: positions L + depth must stay below
  pa.kv = di.kv;
  pa.context_len = di.context_len;
  pa.root_token = di.root_token;
  pa.node_offset = di.node_offset;
  pa.parent = di.parent;
  pa.token = di.token;
  pa.cache_len = pool->cache_len;
  pa.capacity = pool->capacity;
  pa.status = dout.status;
  pa.req_L = (int*)P(w.req_L);
  pa.req_h = (int*)P(w.req_h);
  pa.req_row0 = (int*)P(w.req_row0);
  pa.req_S = (int*)P(w.req_S);
  pa.row_tok = (int*)P(w.row_tok);
  pa.row_pos = (int*)P(w.row_pos);
  pa.row_req = (int*)P(w.row_req);
  pa.row_slot = (int*)P(w.row_slot);
  pa.row_anc = (uint64_t*)P(w.row_anc);
  { KTimer _t(K_PREP, st); CK(prep_launch(pa, st, &launches)); }

  float* X = (float*)P(w.X);
  bf16* Hn = (bf16*)P(w.Hn);
  f16* Q = (f16*)P(w.Q);
  bf16* O = (bf16*)P(w.O);
  bf16* Mb = (bf16*)P(w.M);
  f16* tree_kv = (f16*)P(w.tree_kv);
  // tensor parallel: rank k owns residual rows [k*Rl, k*Rl + nloc) (sequence-parallel residual
  // stream: RMSNorm runs on 1/tp of the rows, C1/C2 become reduce-scatter + bf16 all-gather)
  const bool tp = m->tp_size > 1;
  const int Rl = tp ? (R + m->tp_size - 1) / m->tp_size : R;
  const int r0 = tp ? m->tp_rank * Rl : 0;
  const int nloc = std::max(0, std::min(Rl, R - r0));
  { KTimer _t(K_EMBED, st); if (nloc) CK(embed_launch(m->embed, pa.row_tok + r0, X + (size_t)r0 * c.d, nloc, c.d, st, &launches)); }

  const int hd = c.head_dim, H = c.n_heads, KV = c.n_kv, G = H / KV;
  const int max_pages = (in->max_context_len + 63) / 64;
  AttnArgs aa{};
  aa.Q = Q;
  aa.pool = pool->pages;
  aa.block_table = pool->block_table;
  aa.max_pages_per_seq = pool->max_pages_per_seq;
  aa.num_pages = pool->num_pages;
  aa.tree_kv = tree_kv;
  aa.R_cap = R_cap;
  aa.H = H;
  aa.KV = KV;
  aa.G = G;
  aa.hd = hd;
  aa.req_L = pa.req_L;
  aa.req_h = pa.req_h;
  aa.req_row0 = pa.req_row0;
  aa.req_S = pa.req_S;
  aa.row_anc = pa.row_anc;
  const bool use_tc = attention_tc_supported(hd, G);
  aa.B = B;
  if (use_tc && attn_balanced(max_pages)) {   // persistent grid, even split of all (r, g) sub-tiles
    aa.per_req = 2;
    aa.row_req = pa.row_req;
    aa.nch_tab = (int*)P(w.attn_nch);
    // in-kernel merge when a (request, kv head) has at most one 128-row M-tile (cfg5: 85 rows);
    // bigger groups (cfg4: 520 rows) would stall the merging CTA's pipeline -> combine kernel
    static const int merge_rows = getenv("SPECEDGE_ATTN_MERGE_ROWS") ? atoi(getenv("SPECEDGE_ATTN_MERGE_ROWS")) : 128;
    if ((in->max_nodes + 1) * G <= merge_rows) {
      aa.merge_cnt = (int*)P(w.attn_cnt);
      CK(cudaMemsetAsync(aa.merge_cnt, 0, sizeof(int) * (size_t)B * KV, st));   // self-resetting after
    }
    aa.grid_ctas = num_sms();
    aa.pages_per_split = std::max(1, (max_pages + kMaxSplits - 1) / kMaxSplits);   // unused by the kernel
  } else if (use_tc) {   // per-request chunks (attn_pick_chunk_tc caps them at 8 = kMaxSplits)
    aa.pages_per_split = attn_pick_chunk_tc(B, KV, max_pages);
    aa.per_req = 1;
    aa.row_req = pa.row_req;
  } else {
    aa.n_splits = std::min(kMaxSplits, attn_pick_splits(B, KV, max_pages));
    aa.pages_per_split = std::max(1, (max_pages + aa.n_splits - 1) / aa.n_splits);
  }
  aa.n_splits = aa.per_req == 2 ? kMaxSplits : std::max(1, (max_pages + aa.pages_per_split - 1) / aa.pages_per_split);
  if (aa.n_splits > kMaxSplits) return SPECEDGE_E_UNSUPPORTED;
  aa.max_rows = (in->max_nodes + 1) * G;
  aa.opart = (float*)P(w.opart);
  aa.mpart = (float*)P(w.mpart);
  aa.lpart = (float*)P(w.lpart);
  aa.R = R;
  aa.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)hd));

  if (!tp) CK(cudaMemsetAsync(P(w.tile_cnt), 0, w.tile_cnt_bytes, st));   // fused residual-add counters
  float* Y = (float*)P(w.Y);
  const size_t y_stride = ((size_t)R + kMaxTp) * std::max((H + 2 * KV) * hd, c.d);
  int pendingY = 0;   // K-split partials of the last down-proj not yet added to X
  // row_parallel: O / down under TP -> one unsplit fp32 partial, reduce-scattered over ranks (C1/C2)
  auto f32_gemm = [&](int kind, const CUtensorMap& tm, const void* Xin, int Mrows, int K, bool row_parallel) -> int {
    GemmArgs g{};
    g.M = Mrows;
    g.R = R;
    g.K = K;
    g.out_f32 = Y;
    g.ldo = Mrows;
    g.max_splits = (tp && row_parallel) ? 1 : kind_splits(kind);
    // QKV: its partials are summed by the RoPE kernel; a full wave needs no split (cfg2: 72 pair
    // tiles on 74 pairs -> QKV + RoPE 1.42 -> 1.31 ms per step)
    g.unsplit_if_full = kind == K_QKV ? 1 : 0;
    g.split_stride = y_stride;
    // O / down without tensor parallelism, SPECEDGE_RESID_FUSE bit 0 (O) / bit 1 (down): the residual
    // add (and the K-split sum) happens in the GEMM (GemmArgs::resid) and the next RMSNorm reads X
    // only.  Off by default: measured on cfg2 the epilogue's global read-modify-write of X costs
    // more than the RMSNorm saves (O 0.85 -> 2.05 ms, down 1.66 -> 2.48 ms vs RMSNorm 0.97 -> 0.56
    // ms per step; profiles/README.md)
    static const int resid_fuse = getenv("SPECEDGE_RESID_FUSE") ? atoi(getenv("SPECEDGE_RESID_FUSE")) : 0;
    const bool fuse = !tp && ((kind == K_O && (resid_fuse & 1)) || (kind == K_DOWN && (resid_fuse & 2)));
    if (fuse) {
      g.resid = X;
      g.tile_cnt = (int*)P(w.tile_cnt);
    }
    {
      KTimer _t(kind, st);
      if (gemm_launch(EPI_F32, tm, Xin, g, st, &launches) != cudaSuccess) return -1;
    }
    const int ns = fuse ? 0 : gemm_splits_last();
    if (tp && row_parallel) {
      if (tp_reduce_scatter_f32(Y, (size_t)Rl * Mrows, m->tp_rank, m->nccl, st) != cudaSuccess) return -1;
      ++launches;
    }
    return ns;
  };
  // NEXT-F4: row-parallel GEMM into this rank's peer-mapped output buffer, then the epoch
  // signal; the owner's norm_rows waits and reads its rows from every rank's buffer (tp.cu)
  // Two variants (SPECEDGE_TP_F4=push|pull, default push): push = the GEMM epilogue sends each
  // row to its owner's receive slot with bulk async copies (transfer overlapped with the GEMM);
  // pull = the GEMM writes locally and the owner's RMSNorm loads its rows from every rank.
  const bool fused = tp && m->tp_fused_rows >= R && m->tp_size <= kMaxFusedTp;
  static const bool f4_pull = getenv("SPECEDGE_TP_F4") && std::string(getenv("SPECEDGE_TP_F4")) == "pull";
  bool fused_pending = false;   // a row-parallel partial is waiting in the ranks' buffers
  const float* push_src = nullptr;   // push: the receive buffer holding this rank's tp slots
  const float* nvls_src = nullptr;   // NVLS: multicast address of the pending partial (all rows)
  auto f32_gemm_fused = [&](int kind, const CUtensorMap& tm, const void* Xin, int Mrows, int K) -> int {
    GemmArgs g{};
    g.M = Mrows;
    g.R = R;
    g.K = K;
    g.out_f32 = m->tp_recv;
    g.ldo = Mrows;
    g.max_splits = 1;
    g.split_stride = 0;
    if (m->tp_nvls) {
      // NVLS: the partial goes to this rank's own half of the multicast-bound buffer
      const size_t boff = (size_t)m->tp_fused_buf * m->tp_nvls_buf;
      g.out_f32 = m->tp_nvls_uc + boff;
      nvls_src = m->tp_nvls_mc + boff;
      m->tp_fused_buf ^= 1;
    } else if (!f4_pull) {
      const size_t boff = (size_t)m->tp_fused_buf * m->tp_size * m->tp_fused_slot;
      g.push = 1;
      g.tp_src = m->tp_rank;
      g.rows_per_rank = Rl;
      g.slot_stride = m->tp_fused_slot;
      for (int p = 0; p < m->tp_size; ++p) g.peer_out[p] = m->tp_peer_recv[p] + boff;
      push_src = m->tp_recv + boff;
      m->tp_fused_buf ^= 1;
    }
    {
      KTimer _t(kind, st);
      if (gemm_launch(EPI_F32, tm, Xin, g, st, &launches) != cudaSuccess) return -1;
    }
    if (tp_fused_signal(m, st, &launches) != cudaSuccess) return -1;
    fused_pending = true;
    return m->tp_size;
  };
  // residual add + RMSNorm of this rank's rows (all rows when tp_size == 1), then under TP the
  // bf16 all-gather of the normalised rows for the next column-parallel GEMM
  auto norm_rows = [&](int nY, const bf16* gain, bf16* out, int split) -> specedge_status {
    // NEXT-F4 all-gather (per-layer norms, SPECEDGE_TP_F4_AG=1): every rank stores its normalised
    // rows straight into every rank's copy of Hn (m->tp_hn), then signal + wait replace the NCCL
    // all-gather.  Off by default: measured at parity with NCCL on cfg4 TP=4 (the RMSNorm's remote
    // stores cost what the all-gather did)
    static const bool f4_ag = getenv("SPECEDGE_TP_F4_AG") && getenv("SPECEDGE_TP_F4_AG")[0] == '1';
    const bool ag_fused = fused && f4_ag && !split;
    const bool partial = fused_pending;
    RmsSrc ys{};
    int nYf = nY;
    if (partial && nvls_src) {   // NVLS: the rank sum of this rank's rows in one multimem load
      CK(tp_fused_wait(m, st, &launches));
      ys.mc = nvls_src + (size_t)r0 * c.d;
      nYf = 1;
    } else if (partial) {   // this rank's rows of every rank's partial, summed in rank order
      CK(tp_fused_wait(m, st, &launches));
      for (int p = 0; p < m->tp_size; ++p)
        ys.p[p] = push_src ? push_src + (size_t)p * m->tp_fused_slot
                           : (p == m->tp_rank ? m->tp_recv : m->tp_peer_recv[p]) + (size_t)r0 * c.d;
    }
    if (ag_fused) {
      ys.nout = m->tp_size;
      for (int p = 0; p < m->tp_size; ++p)
        ys.outp[p] = (p == m->tp_rank ? m->tp_hn : m->tp_peer_hn[p]) + (size_t)r0 * c.d;
    }
    {
      KTimer _t(K_RMSNORM, st);
      if (nloc)
        CK(rmsnorm_launch(X + (size_t)r0 * c.d, partial ? nullptr : Y + (size_t)r0 * c.d, nYf, partial ? 0 : y_stride,
                          gain, out + (size_t)(split ? 2 : 1) * r0 * c.d, nloc, c.d, c.eps, st, &launches, split,
                          (partial || ag_fused) ? &ys : nullptr));
    }
    fused_pending = false;
    push_src = nullptr;
    nvls_src = nullptr;
    if (ag_fused) {
      CK(tp_fused_signal(m, st, &launches));
      CK(tp_fused_wait(m, st, &launches));
    } else if (tp) {
      CK(tp_all_gather_bf16(out, (size_t)(split ? 2 : 1) * Rl * c.d, m->tp_rank, m->nccl, st));
      ++launches;
    }
    return SPECEDGE_OK;
  };
  static const bool f4_ag_on = getenv("SPECEDGE_TP_F4_AG") && getenv("SPECEDGE_TP_F4_AG")[0] == '1';
  bf16* const Hn_in = (fused && f4_ag_on) ? m->tp_hn : Hn;   // operand of the column-parallel GEMMs
  // QKV GEMM with the RoPE epilogue (head_dim 128, when gemm_qkv_fused_ok; off with
  // SPECEDGE_QKV_FUSED=0, forced with =2).  Measured on cfg2: 1.13-1.16 ms per step vs 1.00 + 0.35 ms with the
  // fp32 round trip and the separate RoPE kernel (the epilogue stores 16 B per lane after a
  // shared-memory transpose; with 2-B scattered stores it was 1.57 ms)
  static const int qkv_fuse_env = getenv("SPECEDGE_QKV_FUSED") ? atoi(getenv("SPECEDGE_QKV_FUSED")) : 1;
  const bool qkv_fused = qkv_fuse_env > 0 && hd == 128 && (qkv_fuse_env == 2 || gemm_qkv_fused_ok((H + 2 * KV) * hd, R));
  for (int l = 0; l < c.n_layers; ++l) {
    g_dbg_layer = l;
    const auto& Lw = m->layers[l];
    { const specedge_status ns = norm_rows(pendingY, Lw.g_attn, Hn, 0); if (ns != SPECEDGE_OK) return ns; }
    if (qkv_fused) {
      // a4 with RoPE in the GEMM epilogue: q -> Q, k / v -> tree K/V, no fp32 round trip
      GemmArgs gq{};
      gq.M = (H + 2 * KV) * hd;
      gq.R = R;
      gq.K = c.d;
      gq.out_bf16 = reinterpret_cast<bf16*>(Q);
      gq.tree_kv = reinterpret_cast<bf16*>(tree_kv);
      gq.R_cap = R_cap;
      gq.layer = l;
      gq.n_heads = H;
      gq.n_kv = KV;
      gq.head_dim = hd;
      gq.row_pos = pa.row_pos;
      gq.rope_cos = m->rope_cos;
      gq.rope_sin = m->rope_sin;
      KTimer _t(K_QKV, st);
      CK(gemm_launch(EPI_QKV, Lw.tm_qkv, Hn_in, gq, st, &launches));
    } else {
      const int sq = f32_gemm(K_QKV, Lw.tm_qkv, Hn_in, (H + 2 * KV) * hd, c.d, false);
      if (sq < 0) return SPECEDGE_E_CUDA;
      RopeArgs ra{};
      ra.Y = Y;
      ra.nY = sq;
      ra.y_stride = y_stride;
      ra.R = R;
      ra.H = H;
      ra.KV = KV;
      ra.hd = hd;
      ra.layer = l;
      ra.R_cap = R_cap;
      ra.row_pos = pa.row_pos;
      ra.rope_cos = m->rope_cos;
      ra.rope_sin = m->rope_sin;
      ra.Q = Q;
      ra.tree_kv = tree_kv;
      { KTimer _t(K_ROPE, st); CK(qkv_rope_launch(ra, st, &launches)); }
    }
    aa.layer = l;
    if (use_tc) {
      { KTimer _t(K_ATTN, st); CK(attention_tc_launch(aa, B, O, nullptr, st, &launches)); }
      // balanced mode merges its chunks inside the attention kernel (last CTA per (r, g))
      if (aa.n_splits > 1 && !(aa.per_req == 2 && aa.merge_cnt)) { KTimer _t(K_COMBINE, st); CK(attn_combine_launch(aa, O, nullptr, st, &launches)); }
    } else {
      { KTimer _t(K_ATTN, st); CK(attention_launch(aa, B, st, &launches)); }
      { KTimer _t(K_COMBINE, st); CK(attn_combine_launch(aa, O, nullptr, st, &launches)); }
    }
    const int so = fused ? f32_gemm_fused(K_O, Lw.tm_o, O, c.d, H * hd) : f32_gemm(K_O, Lw.tm_o, O, c.d, H * hd, true);
    if (so < 0) return SPECEDGE_E_CUDA;
    { const specedge_status ns = norm_rows(so, Lw.g_mlp, Hn, 0); if (ns != SPECEDGE_OK) return ns; }
    GemmArgs gu{};
    gu.M = 2 * c.ffn;
    gu.R = R;
    gu.K = c.d;
    gu.out_bf16 = Mb;
    gu.ld_out = c.ffn;
    static const int bn_gu = getenv("SPECEDGE_BN_GATEUP") ? atoi(getenv("SPECEDGE_BN_GATEUP")) : 0;
    gu.bn_override = bn_gu;
    if (!tp) {   // last-wave K-parts of the gate/up GEMM go through Y (free between a6's norm and a8)
      gu.tail_buf = Y;
      gu.tail_cap = 4 * (size_t)kGemmSplits * ((size_t)R + kMaxTp) * std::max((size_t)(H + 2 * KV) * hd, (size_t)c.d);
      gu.tile_cnt = (int*)P(w.tile_cnt);
    }
    { KTimer _t(K_GU, st); CK(gemm_launch(EPI_SWIGLU, Lw.tm_gu, Hn_in, gu, st, &launches)); }
    pendingY = fused ? f32_gemm_fused(K_DOWN, Lw.tm_d, Mb, c.d, c.ffn) : f32_gemm(K_DOWN, Lw.tm_d, Mb, c.d, c.ffn, true);
    if (pendingY < 0) return SPECEDGE_E_CUDA;
  }
  int* y = (int*)P(w.y);
  if (!prefill) {
    bf16* Hf = (bf16*)P(w.Hf);
    { const specedge_status ns = norm_rows(pendingY, m->g_final, Hf, 1); if (ns != SPECEDGE_OK) return ns; }
    if (hidden_only) {
      g_last_launches = launches;
      return SPECEDGE_OK;
    }
    GemmArgs gl{};
    gl.M = m->vl;   // this rank's vocab shard (all of V when tp_size == 1)
    gl.R = 2 * R;
    gl.pair = 1;
    gl.K = c.d;
    gl.part_val = (float*)P(w.part_val);
    gl.part_idx = (int*)P(w.part_idx);
    gl.vocab = m->vl;
    gl.vocab_off = m->v0;
    const bool sample = in->mode == SPECEDGE_SAMPLE_TREE && in->temperature >= 1e-6f;
    gl.sample = sample ? 1 : 0;
    gl.inv_t = sample ? (float)(1.0 / (double)in->temperature) : 1.0f;
    gl.seed_lo = (uint32_t)in->seed;
    gl.seed_hi = (uint32_t)(in->seed >> 32);
    gl.row_req = pa.row_req;
    gl.row_slot = pa.row_slot;
    gl.req_round = di.round;
    gl.req_session = di.session_id;
    if (in->mode == SPECEDGE_SAMPLE_PQ_DENSE) {
      // NEXT-F2: pass 1 = Gumbel-max of l/T (bonus after full acceptance) + tile (max, sum exp);
      // pass 2 = p(child) and the Gumbel-max of log max(0, p - q) (bonus after a rejection)
      const int vt = (m->vl + 127) / 128;
      PqArgs pq{};
      pq.B = B;
      pq.R = R;
      pq.ntiles = vt;
      pq.V = c.vocab;
      pq.status = dout.status;
      pq.node_offset = di.node_offset;
      pq.parent = di.parent;
      pq.token = di.token;
      pq.draft_q = in->draft_q;
      pq.row_req = pa.row_req;
      pq.row_slot = pa.row_slot;
      pq.part_m = (float*)P(w.part_m);
      pq.part_s = (float*)P(w.part_s);
      pq.lse = (float*)P(w.lse);
      pq.row_qnode = (int*)P(w.row_qnode);
      pq.pchild = (float*)P(w.pchild);
      pq.y = y;
      pq.resid_y = (int*)P(w.resid_y);
      pq.seed_lo = gl.seed_lo;
      pq.seed_hi = gl.seed_hi;
      pq.req_round = di.round;
      pq.req_session = di.session_id;
      pq.accepted_len = dout.accepted_len;
      pq.accepted_token = dout.accepted_token;
      pq.accepted_node = dout.accepted_node;
      pq.bonus = dout.bonus;
      gl.inv_t = (float)(1.0 / (double)in->temperature);
      GemmArgs g1 = gl;
      g1.sample = 1;
      g1.part_m = (float*)pq.part_m;
      g1.part_s = (float*)pq.part_s;
      { KTimer _t(K_LM, st); CK(gemm_launch(EPI_PQ1, m->tm_lm, Hf, g1, st, &launches)); }
      {
        KTimer _tr(K_LMRED, st);
        CK(lm_reduce_launch(gl.part_val, gl.part_idx, R, vt, y, (float*)P(w.score), dout.row_target, dout.row_score,
                            st, &launches));
        CK(pq_lse_launch(pq, st, &launches));
      }
      GemmArgs g2 = gl;
      g2.sample = 1;
      g2.lse = pq.lse;
      g2.row_qnode = pq.row_qnode;
      g2.node_token = di.token;
      g2.draft_q = in->draft_q;
      g2.vocab_q = c.vocab;
      g2.pchild = (float*)pq.pchild;
      { KTimer _t(K_LM, st); CK(gemm_launch(EPI_PQ2, m->tm_lm, Hf, g2, st, &launches)); }
      {
        KTimer _tr(K_LMRED, st);
        CK(lm_reduce_launch(gl.part_val, gl.part_idx, R, vt, (int*)P(w.resid_y), (float*)P(w.resid_s), nullptr,
                            nullptr, st, &launches));
      }
      { KTimer _t(K_WALK, st); CK(pq_walk_launch(pq, st, &launches)); }
    } else if (lm_hi_only()) {
      // hi-only LM head (one MMA pass over the vocabulary instead of the hi/lo pair) + exact
      // rescoring of the candidates its window cannot rule out (k_lm_refine, internal.h)
      GemmArgs gh = gl;
      gh.pair = 0;
      gh.R = R;
      gh.x_stride = 2 * c.d;   // the even (hi) rows of the interleaved final hidden
      gh.top2 = 1;
      gh.part_val2 = (float*)P(w.part_val2);
      gh.part_idx2 = (int*)P(w.part_idx2);
      gh.part_val3 = (float*)P(w.part_val3);
      { KTimer _t(K_LM, st); CK(gemm_launch(EPI_ARGMAX, m->tm_lm, Hf, gh, st, &launches)); }
      RefineArgs rf{};
      rf.R = R;
      rf.ntiles = (m->vl + 127) / 128;
      rf.d = c.d;
      rf.vocab = m->vl;
      rf.vocab_off = m->v0;
      rf.sample = gl.sample;
      rf.inv_t = gl.inv_t;
      rf.wmax = m->lm_wmax;
      rf.part_val = gl.part_val;
      rf.part_idx = gl.part_idx;
      rf.part_val2 = gh.part_val2;
      rf.part_idx2 = gh.part_idx2;
      rf.part_val3 = gh.part_val3;
      rf.hf = Hf;
      rf.w = m->lm_head;
      rf.seed_lo = gl.seed_lo;
      rf.seed_hi = gl.seed_hi;
      rf.row_req = pa.row_req;
      rf.row_slot = pa.row_slot;
      rf.req_round = di.round;
      rf.req_session = di.session_id;
      rf.y = y;
      rf.score = (float*)P(w.score);
      rf.row_target = tp ? nullptr : dout.row_target;
      rf.row_score = tp ? nullptr : dout.row_score;
      KTimer _tr(K_LMRED, st);
      CK(lm_refine_launch(rf, st, &launches));
      if (tp)
        CK(tp_argmax_gather(y, (float*)P(w.score), R, (float*)P(w.tp_gather), m->tp_size, m->nccl, dout.row_target,
                            dout.row_score, st, &launches));
    } else {
      { KTimer _t(K_LM, st); CK(gemm_launch(EPI_ARGMAX, m->tm_lm, Hf, gl, st, &launches)); }
      KTimer _tr(K_LMRED, st);
      CK(lm_reduce_launch(gl.part_val, gl.part_idx, R, (m->vl + 127) / 128, y, (float*)P(w.score),
                          tp ? nullptr : dout.row_target, tp ? nullptr : dout.row_score, st, &launches));
      if (tp)
        CK(tp_argmax_gather(y, (float*)P(w.score), R, (float*)P(w.tp_gather), m->tp_size, m->nccl, dout.row_target,
                            dout.row_score, st, &launches));
    }
  }
  const bool pq_walked = !prefill && in->mode == SPECEDGE_SAMPLE_PQ_DENSE;
  WalkArgs wa{};
  wa.B = B;
  wa.force_chain = prefill ? 1 : 0;
  wa.status = dout.status;
  wa.node_offset = di.node_offset;
  wa.parent = di.parent;
  wa.token = di.token;
  wa.y = y;
  wa.accepted_len = dout.accepted_len;
  wa.accepted_token = dout.accepted_token;
  wa.accepted_node = dout.accepted_node;
  wa.bonus = dout.bonus;
  if (!pq_walked) { KTimer _t(K_WALK, st); CK(walk_launch(wa, st, &launches)); }
  if (do_commit) {
    CommitArgs ca{};
    ca.B = B;
    ca.layers = c.n_layers;
    ca.KV = KV;
    ca.hd = hd;
    ca.R_cap = R_cap;
    ca.num_pages = pool->num_pages;
    ca.max_pages_per_seq = pool->max_pages_per_seq;
    ca.status = dout.status;
    ca.req_L = pa.req_L;
    ca.req_h = pa.req_h;
    ca.req_row0 = pa.req_row0;
    ca.node_offset = di.node_offset;
    ca.accepted_len = dout.accepted_len;
    ca.accepted_node = dout.accepted_node;
    ca.tree_kv = tree_kv;
    ca.pool = pool->pages;
    ca.block_table = pool->block_table;
    ca.cache_len = pool->cache_len;
    KTimer _t(K_COMMIT, st);
    CK(commit_launch(ca, st, &launches));
  }
  g_last_launches = launches;
  return SPECEDGE_OK;
}

specedge_status check_in(const specedge_model* m, const specedge_kvpool* pool, const specedge_verify_in* in) {
  if (!m || !pool || !in) return SPECEDGE_E_INVALID;
  if (pool->model != m) return SPECEDGE_E_INVALID;
  if (in->num_requests <= 0 || in->total_nodes < 0) return SPECEDGE_E_INVALID;
  if (in->max_nodes < 0 || in->max_nodes > SPECEDGE_MAX_NODES) return SPECEDGE_E_INVALID;
  if (in->max_context_len <= 0 || in->max_context_len > m->cfg.max_position) return SPECEDGE_E_INVALID;
  if (in->mode != SPECEDGE_GREEDY && in->mode != SPECEDGE_SAMPLE_TREE && in->mode != SPECEDGE_SAMPLE_PQ_DENSE)
    return SPECEDGE_E_INVALID;
  if (in->mode == SPECEDGE_SAMPLE_TREE && !(in->temperature >= 0.f)) return SPECEDGE_E_INVALID;
  if (in->mode == SPECEDGE_SAMPLE_PQ_DENSE) {
    if (!(in->temperature >= 1e-6f) || (in->total_nodes > 0 && !in->draft_q)) return SPECEDGE_E_INVALID;
    if (m->tp_size != 1) return SPECEDGE_E_UNSUPPORTED;
  }
  if (!in->kv || !in->context_len || !in->root_token || !in->session_id || !in->round || !in->node_offset)
    return SPECEDGE_E_INVALID;
  if (in->total_nodes > 0 && (!in->parent || !in->token)) return SPECEDGE_E_INVALID;
  return SPECEDGE_OK;
}

specedge_status check_out(const specedge_verify_out* out, int total_nodes) {
  if (!out || !out->status || !out->accepted_len || !out->bonus) return SPECEDGE_E_INVALID;
  if (total_nodes > 0 && (!out->accepted_token || !out->accepted_node)) return SPECEDGE_E_INVALID;
  return SPECEDGE_OK;
}

// ---- CUDA-graph replay of whole verify steps -----------------------------------------------
// A verify step is a fixed sequence of ~8 + 8*layers launches whose parameters depend only on the
// host scalars of specedge_verify_in and on buffer addresses.  The first call with a given
// signature records the step (stream capture on a model-owned stream: the caller's stream may be
// the legacy default stream, which cannot be captured) and instantiates it; every call then
// replays it with one cudaGraphLaunch on the caller's stream.
// Disabled by SPECEDGE_NO_GRAPH=1, while kernel timing is on, and when the caller's stream is
// itself being captured (the plain launches then become part of the caller's graph).
bool graphs_enabled(const specedge_model* m, cudaStream_t st) {
  static const bool off = getenv("SPECEDGE_NO_GRAPH") && getenv("SPECEDGE_NO_GRAPH")[0] == '1';
  // tensor parallel: NCCL collectives issued earlier on another stream (prefill) make the capture
  // of the next collective wait on an event from outside the capture on one rank only -> the
  // ranks' collective sequences diverge; TP steps (~100 ms) gain nothing from graph replay anyway
  if (off || g_timing.on || m->tp_size > 1) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return false;
  }
  return true;
}

template <typename F>
specedge_status run_graphed(specedge_model* m, const std::string& key, cudaStream_t st, F&& body) {
  if (!m->gstream) {
    CK(cudaStreamCreateWithFlags(&m->gstream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&m->gev_in, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&m->gev_out, cudaEventDisableTiming));
  }
  cudaGraphExec_t exec = nullptr;
  for (size_t i = 0; i < m->graphs.size(); ++i)
    if (m->graphs[i].key == key) {
      exec = m->graphs[i].exec;
      if (i) std::swap(m->graphs[i], m->graphs[0]);   // most recent first
      break;
    }
  if (exec) {
    ++m->graph_stats[0];
  } else {
    // a signature is captured on its second use: one-off shapes (a serving loop's ragged batches)
    // run as plain launches on the caller's stream instead of paying a capture + instantiation
    auto it = std::find(m->graph_seen.begin(), m->graph_seen.end(), key);
    if (it == m->graph_seen.end()) {
      if (m->graph_seen.size() >= 64) m->graph_seen.erase(m->graph_seen.begin());
      m->graph_seen.push_back(key);
      ++m->graph_stats[2];
      return body(st);
    }
    m->graph_seen.erase(it);
    ++m->graph_stats[1];
    CK(cudaStreamBeginCapture(m->gstream, cudaStreamCaptureModeThreadLocal));
    const specedge_status s = body(m->gstream);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(m->gstream, &graph);
    if (s != SPECEDGE_OK || e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      return s != SPECEDGE_OK ? s : SPECEDGE_E_CUDA;
    }
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(ei);
    if (m->graphs.size() >= 32) {
      cudaGraphExecDestroy(m->graphs.back().exec);
      m->graphs.pop_back();
    }
    m->graphs.insert(m->graphs.begin(), specedge_model::Graph{key, exec});
  }
  // recorded on the model's stream (capture never executes anything), replayed on the caller's
  CK(cudaGraphLaunch(exec, st));
  return SPECEDGE_OK;
}

template <typename... T>
std::string graph_key(const specedge_verify_in* in, T... extra) {
  std::string k;
  auto put = [&](const void* p, size_t n) { k.append(reinterpret_cast<const char*>(p), n); };
  put(&in->num_requests, sizeof(int32_t) * 5);   // num_requests .. mode
  put(&in->temperature, sizeof(float));
  put(&in->seed, sizeof(uint64_t));
  put(&in->auto_commit, sizeof(int32_t));
  (put(&extra, sizeof(extra)), ...);
  return k;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

specedge_status specedge_model_create(const specedge_model_config* cfg, uint64_t weight_seed, int32_t device,
                                      specedge_model** out) {
  return specedge_model_create_tp(cfg, weight_seed, device, 0, 1, nullptr, out);
}

specedge_status specedge_tp_unique_id(uint8_t* id) {
  if (!id) return SPECEDGE_E_INVALID;
  const int r = tp_unique_id(id);
  return r == 0 ? SPECEDGE_OK : (r == -1 ? SPECEDGE_E_UNSUPPORTED : SPECEDGE_E_CUDA);
}

specedge_status specedge_model_create_tp(const specedge_model_config* cfg, uint64_t weight_seed, int32_t device,
                                         int32_t tp_rank, int32_t tp_size, const uint8_t* nccl_id,
                                         specedge_model** out) {
  if (!cfg || !out) return SPECEDGE_E_INVALID;
  if (tp_size < 1 || tp_size > kMaxTp || tp_rank < 0 || tp_rank >= tp_size) return SPECEDGE_E_INVALID;
  // nccl_id == NULL with tp_size > 1: a communicator-less shard (weights, KV pool, introspection;
  // verify / prefill return E_UNSUPPORTED) — lets one process check the sharding on one GPU
  if (!check_cfg(*cfg)) return SPECEDGE_E_UNSUPPORTED;
  // head-parallel attention, column-parallel QKV / gate-up (gate-up in 64-row blocks),
  // row-parallel O / down, vocab-parallel LM head
  if (cfg->n_kv % tp_size || cfg->n_heads % tp_size || cfg->ffn % (64 * tp_size) || cfg->vocab < tp_size)
    return SPECEDGE_E_UNSUPPORTED;
  specedge_model_config lc = *cfg;
  lc.n_heads /= tp_size;
  lc.n_kv /= tp_size;
  lc.ffn /= tp_size;
  if (!check_cfg(lc)) return SPECEDGE_E_UNSUPPORTED;
  if (tp_size > 1 && nccl_id && !tp_available()) return SPECEDGE_E_UNSUPPORTED;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return SPECEDGE_E_DEVICE;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return SPECEDGE_E_DEVICE;
  CK(cudaSetDevice(device));
  specedge_model* m = new specedge_model();
  m->gcfg = *cfg;
  m->cfg = lc;
  m->device = device;
  m->tp_rank = tp_rank;
  m->tp_size = tp_size;
  {
    const int vs = (cfg->vocab + tp_size - 1) / tp_size;
    m->v0 = std::min(cfg->vocab, tp_rank * vs);
    m->vl = std::min(cfg->vocab, m->v0 + vs) - m->v0;
  }
  const auto& c = lc;   // rank-local shapes
  const size_t H = c.n_heads, KV = c.n_kv, hd = c.head_dim, d = c.d, F = c.ffn, V = c.vocab, Vl = m->vl;
  const size_t gH = cfg->n_heads, gF = cfg->ffn;
  const uint32_t k0 = (uint32_t)weight_seed, k1 = (uint32_t)(weight_seed >> 32);
  auto fail = [&](specedge_status s) {
    for (void* p : m->allocs) cudaFree(p);
    if (m->nccl) tp_comm_destroy(m->nccl);
    delete m;
    return s;
  };
  auto sc = [](double stdv) { return (float)(stdv * std::sqrt(3.0) * std::ldexp(1.0, -23)); };
  // off0..2: global row offsets of the local parts, col0/gcols: column shard of the global matrix
  auto init = [&](bf16* dst, long long rows, long long cols, int layout, int t0, int t1, int t2, int layer,
                  long long r0, long long r1, float s0, float s1, float s2, int gain, long long off0 = 0,
                  long long off1 = 0, long long off2 = 0, long long col0 = 0, long long gcols = -1) {
    InitArgs a{};
    a.off0 = off0;
    a.off1 = off1;
    a.off2 = off2;
    a.col0 = col0;
    a.gcols = gcols < 0 ? cols : gcols;
    a.dst = dst;
    a.rows = rows;
    a.cols = cols;
    a.layout = layout;
    a.tid0 = t0;
    a.tid1 = t1;
    a.tid2 = t2;
    a.layer = layer;
    a.rows0 = r0;
    a.rows1 = r1;
    a.scale0 = s0;
    a.scale1 = s1;
    a.scale2 = s2;
    a.gain = gain;
    a.k0 = k0;
    a.k1 = k1;
    return init_weights_launch(a, 0);
  };
  m->embed = dalloc<bf16>(m, V * d);
  m->lm_head = dalloc<bf16>(m, Vl * d);
  m->g_final = dalloc<bf16>(m, d);
  if (!m->embed || !m->lm_head || !m->g_final) return fail(SPECEDGE_E_OOM);
  if (init(m->embed, V, d, INIT_PLAIN, 1, 0, 0, 0, 0, 0, sc(1.0), 0, 0, 0) != cudaSuccess) return fail(SPECEDGE_E_CUDA);
  if (init(m->lm_head, Vl, d, INIT_PLAIN, 9, 0, 0, 0, 0, 0, sc(2.0 / std::sqrt((double)d)), 0, 0, 0, m->v0) != cudaSuccess)
    return fail(SPECEDGE_E_CUDA);
  if (init(m->g_final, 1, d, INIT_PLAIN, 12, 0, 0, 0, 0, 0, 0, 0, 0, 1) != cudaSuccess) return fail(SPECEDGE_E_CUDA);
  m->layers.resize(c.n_layers);
  const double s_d = 1.0 / std::sqrt((double)d), s_q = 1.0 / std::sqrt((double)(gH * hd)), s_f = 1.0 / std::sqrt((double)gF);
  const long long rk = tp_rank;
  for (int l = 0; l < c.n_layers; ++l) {
    auto& L = m->layers[l];
    L.wqkv = dalloc<bf16>(m, (H + 2 * KV) * hd * d);
    L.wo = dalloc<bf16>(m, d * H * hd);
    L.wgu = dalloc<bf16>(m, 2 * F * d);
    L.wd = dalloc<bf16>(m, d * F);
    L.g_attn = dalloc<bf16>(m, d);
    L.g_mlp = dalloc<bf16>(m, d);
    if (!L.wqkv || !L.wo || !L.wgu || !L.wd || !L.g_attn || !L.g_mlp) return fail(SPECEDGE_E_OOM);
    bool ok = init(L.wqkv, (H + 2 * KV) * hd, d, INIT_QKV, 2, 3, 4, l, H * hd, KV * hd, sc(s_d), sc(s_d), sc(s_d), 0,
                   rk * H * hd, rk * KV * hd, rk * KV * hd) == cudaSuccess;
    ok = ok && init(L.wo, d, H * hd, INIT_PLAIN, 5, 0, 0, l, 0, 0, sc(s_q), 0, 0, 0, 0, 0, 0, rk * H * hd,
                    (long long)gH * hd) == cudaSuccess;
    ok = ok && init(L.wgu, 2 * F, d, INIT_GATEUP, 6, 7, 0, l, F, 0, sc(s_d), sc(s_d), 0, 0, rk * F) == cudaSuccess;
    ok = ok && init(L.wd, d, F, INIT_PLAIN, 8, 0, 0, l, 0, 0, sc(s_f), 0, 0, 0, 0, 0, 0, rk * F, (long long)gF) == cudaSuccess;
    ok = ok && init(L.g_attn, 1, d, INIT_PLAIN, 10, 0, 0, l, 0, 0, 0, 0, 0, 1) == cudaSuccess;
    ok = ok && init(L.g_mlp, 1, d, INIT_PLAIN, 11, 0, 0, l, 0, 0, 0, 0, 0, 1) == cudaSuccess;
    if (!ok) return fail(SPECEDGE_E_CUDA);
    ok = make_tmap_2d(&L.tm_qkv, L.wqkv, (H + 2 * KV) * hd, d, 128) && make_tmap_2d(&L.tm_o, L.wo, d, H * hd, 128) &&
         make_tmap_2d(&L.tm_gu, L.wgu, 2 * F, d, 128) && make_tmap_2d(&L.tm_d, L.wd, d, F, 128);
    if (!ok) return fail(SPECEDGE_E_CUDA);
  }
  if (!make_tmap_2d(&m->tm_lm, m->lm_head, Vl, d, 128)) return fail(SPECEDGE_E_CUDA);
  {   // max_v ||W_v||_2 of this shard's LM-head rows: the hi-only LM head's rescoring window
    float* dmax = dalloc<float>(m, 1);
    if (!dmax || row_norm_max_launch(m->lm_head, (int)Vl, (int)d, dmax, 0) != cudaSuccess ||
        cudaMemcpy(&m->lm_wmax, dmax, sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(SPECEDGE_E_CUDA);
    m->lm_wmax *= 1.0001f;   // margin over the fp32 evaluation of the norm
  }
  // RoPE table: angles in double (amb. A14), stored fp32
  const size_t half = hd / 2;
  std::vector<float> cs((size_t)c.max_position * half), sn((size_t)c.max_position * half);
  for (size_t i = 0; i < half; ++i) {
    const double inv = std::pow(c.rope_theta, -2.0 * (double)i / (double)hd);
    for (int p = 0; p < c.max_position; ++p) {
      const double ang = (double)p * inv;
      cs[(size_t)p * half + i] = (float)std::cos(ang);
      sn[(size_t)p * half + i] = (float)std::sin(ang);
    }
  }
  m->rope_cos = dalloc<float>(m, cs.size());
  m->rope_sin = dalloc<float>(m, sn.size());
  if (!m->rope_cos || !m->rope_sin) return fail(SPECEDGE_E_OOM);
  if (cudaMemcpy(m->rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(m->rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(SPECEDGE_E_CUDA);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(SPECEDGE_E_CUDA);
  if (tp_size > 1 && nccl_id && tp_comm_init(&m->nccl, nccl_id, tp_rank, tp_size) != 0) return fail(SPECEDGE_E_CUDA);
  *out = m;
  return SPECEDGE_OK;
}

specedge_status specedge_model_tp_info(const specedge_model* m, int32_t* tp_rank, int32_t* tp_size, int32_t* vocab0,
                                       int32_t* vocab_n) {
  if (!m) return SPECEDGE_E_INVALID;
  if (tp_rank) *tp_rank = m->tp_rank;
  if (tp_size) *tp_size = m->tp_size;
  if (vocab0) *vocab0 = m->v0;
  if (vocab_n) *vocab_n = m->vl;
  return SPECEDGE_OK;
}

specedge_status specedge_tp_fused_enable(specedge_model* m, int32_t max_rows, void* stream) {
  if (!m || m->tp_size < 2 || m->tp_size > kMaxFusedTp || max_rows <= 0) return SPECEDGE_E_INVALID;
  CK(cudaSetDevice(m->device));
  const int r = tp_fused_enable(m, max_rows, (cudaStream_t)stream);
  if (r == 0) return SPECEDGE_OK;
  if (r == -1 || r == -2) return SPECEDGE_E_INVALID;
  m->tp_fused_rows = 0;
  return SPECEDGE_E_CUDA;
}

int32_t specedge_tp_fused_mode(const specedge_model* m) {
  if (!m || !m->tp_fused_rows) return 0;
  if (m->tp_nvls) return 3;
  static const bool f4_pull = getenv("SPECEDGE_TP_F4") && std::string(getenv("SPECEDGE_TP_F4")) == "pull";
  return f4_pull ? 2 : 1;
}

specedge_status specedge_model_destroy(specedge_model* m) {
  if (!m) return SPECEDGE_E_INVALID;
  cudaSetDevice(m->device);
  cudaDeviceSynchronize();
  tp_fused_close(m);
  if (m->nccl) tp_comm_destroy(m->nccl);
  for (auto& g : m->graphs) cudaGraphExecDestroy(g.exec);
  if (m->gstream) cudaStreamDestroy(m->gstream);
  if (m->gev_in) cudaEventDestroy(m->gev_in);
  if (m->gev_out) cudaEventDestroy(m->gev_out);
  if (m->pinned) cudaFreeHost(m->pinned);
  for (void* p : m->allocs) cudaFree(p);
  delete m;
  return SPECEDGE_OK;
}

specedge_status specedge_kvpool_create(specedge_model* m, int32_t num_pages, int32_t max_handles, specedge_kvpool** out) {
  if (!m || !out || num_pages <= 0 || max_handles <= 0) return SPECEDGE_E_INVALID;
  CK(cudaSetDevice(m->device));
  const auto& c = m->cfg;
  specedge_kvpool* p = new specedge_kvpool();
  p->model = m;
  p->num_pages = num_pages;
  p->max_handles = max_handles;
  p->max_pages_per_seq = (c.max_position + kPage - 1) / kPage;
  const size_t page_elems = (size_t)c.n_layers * 2 * c.n_kv * kPage * c.head_dim;
  bool ok = cudaMalloc(&p->pages, page_elems * num_pages * sizeof(bf16)) == cudaSuccess;
  ok = ok && cudaMalloc(&p->block_table, sizeof(int) * (size_t)max_handles * p->max_pages_per_seq) == cudaSuccess;
  ok = ok && cudaMalloc(&p->cache_len, sizeof(int) * max_handles) == cudaSuccess;
  ok = ok && cudaMalloc(&p->capacity, sizeof(int) * max_handles) == cudaSuccess;
  if (!ok) {
    cudaFree(p->pages);
    cudaFree(p->block_table);
    cudaFree(p->cache_len);
    cudaFree(p->capacity);
    delete p;
    return SPECEDGE_E_OOM;
  }
  CK(cudaMemset(p->pages, 0, page_elems * num_pages * sizeof(bf16)));
  CK(cudaMemset(p->block_table, 0, sizeof(int) * (size_t)max_handles * p->max_pages_per_seq));
  CK(cudaMemset(p->cache_len, 0, sizeof(int) * max_handles));
  CK(cudaMemset(p->capacity, 0, sizeof(int) * max_handles));
  CK(cudaDeviceSynchronize());
  p->free_pages.resize(num_pages);
  for (int i = 0; i < num_pages; ++i) p->free_pages[i] = num_pages - 1 - i;
  p->handle_pages.resize(max_handles);
  p->handle_cap.assign(max_handles, 0);
  *out = p;
  return SPECEDGE_OK;
}

specedge_status specedge_kvpool_destroy(specedge_kvpool* p) {
  if (!p) return SPECEDGE_E_INVALID;
  cudaSetDevice(p->model->device);
  cudaFree(p->pages);
  cudaFree(p->block_table);
  cudaFree(p->cache_len);
  cudaFree(p->capacity);
  delete p;
  return SPECEDGE_OK;
}

specedge_status specedge_kv_alloc(specedge_kvpool* p, int32_t capacity_tokens, int32_t* out_handle) {
  if (!p || !out_handle || capacity_tokens <= 0) return SPECEDGE_E_INVALID;
  const int need = (capacity_tokens + kPage - 1) / kPage;
  if (need > p->max_pages_per_seq || capacity_tokens > p->model->cfg.max_position) return SPECEDGE_E_INVALID;
  int h = -1;
  for (int i = 0; i < p->max_handles; ++i)
    if (p->handle_cap[i] == 0) { h = i; break; }
  if (h < 0 || (int)p->free_pages.size() < need) return SPECEDGE_E_OOM;
  std::vector<int> pages(need);
  for (int i = 0; i < need; ++i) {
    pages[i] = p->free_pages.back();
    p->free_pages.pop_back();
  }
  CK(cudaSetDevice(p->model->device));
  CK(cudaMemcpy(p->block_table + (size_t)h * p->max_pages_per_seq, pages.data(), need * sizeof(int), cudaMemcpyHostToDevice));
  const int zero = 0;
  CK(cudaMemcpy(p->cache_len + h, &zero, sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(p->capacity + h, &capacity_tokens, sizeof(int), cudaMemcpyHostToDevice));
  p->handle_pages[h] = pages;
  p->handle_cap[h] = capacity_tokens;
  *out_handle = h;
  return SPECEDGE_OK;
}

specedge_status specedge_kv_free(specedge_kvpool* p, int32_t h) {
  if (!p || h < 0 || h >= p->max_handles || p->handle_cap[h] == 0) return SPECEDGE_E_INVALID;
  for (int pg : p->handle_pages[h]) p->free_pages.push_back(pg);
  p->handle_pages[h].clear();
  p->handle_cap[h] = 0;
  const int zero = 0;
  CK(cudaSetDevice(p->model->device));
  CK(cudaMemcpy(p->capacity + h, &zero, sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(p->cache_len + h, &zero, sizeof(int), cudaMemcpyHostToDevice));
  return SPECEDGE_OK;
}

specedge_status specedge_kv_set_len(specedge_kvpool* p, const int32_t* handles, const int32_t* lens, int32_t n, void* stream) {
  if (!p || !handles || !lens || n < 0) return SPECEDGE_E_INVALID;
  for (int i = 0; i < n; ++i) {
    const int h = handles[i];
    if (h < 0 || h >= p->max_handles || p->handle_cap[h] == 0 || lens[i] < 0 || lens[i] > p->handle_cap[h])
      return SPECEDGE_E_INVALID;
  }
  // lengths travel as kernel parameters (stream-ordered, graph-capturable, no host staging)
  for (int i0 = 0; i0 < n; i0 += kSetLenBatch) {
    SetLenArgs a{};
    a.n = std::min(kSetLenBatch, n - i0);
    for (int i = 0; i < a.n; ++i) {
      a.handle[i] = handles[i0 + i];
      a.len[i] = lens[i0 + i];
    }
    CK(set_len_launch(p->cache_len, a, (cudaStream_t)stream));
  }
  return SPECEDGE_OK;
}

specedge_status specedge_kv_get_len(specedge_kvpool* p, const int32_t* handles, int32_t* lens, int32_t n) {
  if (!p || !handles || !lens || n < 0) return SPECEDGE_E_INVALID;
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < n; ++i) {
    const int h = handles[i];
    if (h < 0 || h >= p->max_handles) return SPECEDGE_E_INVALID;
    CK(cudaMemcpy(lens + i, p->cache_len + h, sizeof(int), cudaMemcpyDeviceToHost));
  }
  return SPECEDGE_OK;
}

specedge_status specedge_kv_fill_random(specedge_kvpool* p, int32_t h, int32_t n_tokens, uint64_t seed, uint32_t stream_id,
                                        void* stream) {
  if (!p || h < 0 || h >= p->max_handles || p->handle_cap[h] == 0 || n_tokens < 0 || n_tokens > p->handle_cap[h])
    return SPECEDGE_E_INVALID;
  const auto& c = p->model->cfg;
  CK(kv_fill_launch(p->pages, p->block_table + (size_t)h * p->max_pages_per_seq, c.n_layers, p->num_pages, c.n_kv,
                    c.head_dim, n_tokens, (uint32_t)seed, (uint32_t)(seed >> 32), stream_id, p->model->tp_rank * c.n_kv,
                    (cudaStream_t)stream));
  CK(cudaMemcpyAsync(p->cache_len + h, &n_tokens, sizeof(int), cudaMemcpyHostToDevice, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return SPECEDGE_OK;
}

specedge_status specedge_workspace_size(const specedge_model* m, int32_t max_requests, int32_t max_rows,
                                        int32_t max_context_len, size_t* bytes) {
  if (!m || !bytes || max_requests <= 0 || max_rows < max_requests || max_context_len <= 0) return SPECEDGE_E_INVALID;
  *bytes = ws_layout(m->cfg, max_requests, max_rows).total;
  return SPECEDGE_OK;
}


specedge_status specedge_verify_batch(specedge_model* m, specedge_kvpool* pool, const specedge_verify_in* in,
                                      specedge_verify_out* out, void* workspace, size_t ws_bytes, void* stream) {
  specedge_status s = check_in(m, pool, in);
  if (s != SPECEDGE_OK) return s;
  if ((s = check_out(out, in->total_nodes)) != SPECEDGE_OK) return s;
  DevIn di{in->kv, in->context_len, in->root_token, in->node_offset, in->parent, in->token, in->session_id, in->round};
  DevOut dout{out->status, out->accepted_len, out->accepted_token, out->accepted_node, out->bonus, out->row_target,
              out->row_score};
  const cudaStream_t st = (cudaStream_t)stream;
  if (!graphs_enabled(m, st))
    return run_verify(m, pool, in, di, dout, (uint8_t*)workspace, ws_bytes, st, false, in->auto_commit != 0);
  const std::string key = graph_key(in, (const void*)pool, workspace, ws_bytes, (const void*)in->kv,
                                    (const void*)in->context_len, (const void*)in->root_token,
                                    (const void*)in->node_offset, (const void*)in->parent, (const void*)in->token,
                                    (const void*)in->session_id, (const void*)in->round, (const void*)out->status,
                                    (const void*)out->accepted_len, (const void*)out->accepted_token,
                                    (const void*)out->accepted_node, (const void*)out->bonus,
                                    (const void*)out->row_target, (const void*)out->row_score,
                                    (const void*)in->draft_q, 1);
  return run_graphed(m, key, st, [&](cudaStream_t gs) {
    return run_verify(m, pool, in, di, dout, (uint8_t*)workspace, ws_bytes, gs, false, in->auto_commit != 0);
  });
}

specedge_status specedge_graph_stats(const specedge_model* m, int64_t* out3, int32_t reset) {
  if (!m || !out3) return SPECEDGE_E_INVALID;
  for (int i = 0; i < 3; ++i) out3[i] = m->graph_stats[i];
  if (reset) for (int i = 0; i < 3; ++i) const_cast<specedge_model*>(m)->graph_stats[i] = 0;
  return SPECEDGE_OK;
}

specedge_status specedge_kv_commit(specedge_model* m, specedge_kvpool* pool, const specedge_verify_in* in,
                                   specedge_verify_out* out, void* workspace, size_t ws_bytes, void* stream) {
  specedge_status s = check_in(m, pool, in);
  if (s != SPECEDGE_OK) return s;
  if ((s = check_out(out, in->total_nodes)) != SPECEDGE_OK) return s;
  const auto& c = m->cfg;
  const int B = in->num_requests, R = in->total_nodes + B;
  const WsLayout w = ws_layout(c, B, R);
  if (!workspace || ws_bytes < w.total) return SPECEDGE_E_WORKSPACE;
  uint8_t* ws = (uint8_t*)workspace;
  CommitArgs ca{};
  ca.B = B;
  ca.layers = c.n_layers;
  ca.KV = c.n_kv;
  ca.hd = c.head_dim;
  ca.R_cap = R;
  ca.num_pages = pool->num_pages;
  ca.max_pages_per_seq = pool->max_pages_per_seq;
  ca.status = out->status;
  ca.req_L = (int*)(ws + w.req_L);
  ca.req_h = (int*)(ws + w.req_h);
  ca.req_row0 = (int*)(ws + w.req_row0);
  ca.node_offset = in->node_offset;
  ca.accepted_len = out->accepted_len;
  ca.accepted_node = out->accepted_node;
  ca.tree_kv = (f16*)(ws + w.tree_kv);
  ca.pool = pool->pages;
  ca.block_table = pool->block_table;
  ca.cache_len = pool->cache_len;
  int launches = 0;
  CK(commit_launch(ca, (cudaStream_t)stream, &launches));
  return SPECEDGE_OK;
}

specedge_status specedge_verify_batch_host(specedge_model* m, specedge_kvpool* pool, const specedge_verify_in* in,
                                           specedge_verify_out* out, void* workspace, size_t ws_bytes, void* stream) {
  specedge_status s = check_in(m, pool, in);
  if (s != SPECEDGE_OK) return s;
  if (in->mode == SPECEDGE_SAMPLE_PQ_DENSE) return SPECEDGE_E_UNSUPPORTED;   // dense q: device entry only
  if ((s = check_out(out, in->total_nodes)) != SPECEDGE_OK) return s;
  const auto& c = m->cfg;
  const int B = in->num_requests, T = in->total_nodes, R = T + B;
  const WsLayout w = ws_layout(c, B, R);
  if (!workspace || ws_bytes < w.total) return SPECEDGE_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  // pack inputs into one pinned block -> one H2D copy
  auto a8 = [](size_t x) { return (x + 7) & ~size_t(7); };
  size_t o_kv = 0, o_ctx = a8(o_kv + 4 * B), o_root = a8(o_ctx + 4 * B), o_round = a8(o_root + 4 * B),
         o_ses = a8(o_round + 4 * B), o_off = a8(o_ses + 8 * B), o_par = a8(o_off + 4 * (B + 1)),
         o_tok = a8(o_par + 4 * T), in_bytes = a8(o_tok + 4 * T);
  size_t q_st = 0, q_al = a8(4 * B), q_bo = a8(q_al + 4 * B), q_at = a8(q_bo + 4 * B), q_an = a8(q_at + 4 * T),
         q_rt = a8(q_an + 4 * T), q_rs = a8(q_rt + 4 * R), out_bytes = a8(q_rs + 4 * R);
  const size_t need = in_bytes + out_bytes;
  if (m->pinned_bytes < need) {
    if (m->pinned) cudaFreeHost(m->pinned);
    m->pinned = nullptr;
    m->pinned_bytes = 0;
    CK(cudaHostAlloc(&m->pinned, need * 2, cudaHostAllocDefault));
    m->pinned_bytes = need * 2;
  }
  uint8_t* hb = (uint8_t*)m->pinned;
  std::memcpy(hb + o_kv, in->kv, 4 * B);
  std::memcpy(hb + o_ctx, in->context_len, 4 * B);
  std::memcpy(hb + o_root, in->root_token, 4 * B);
  std::memcpy(hb + o_round, in->round, 4 * B);
  std::memcpy(hb + o_ses, in->session_id, 8 * B);
  std::memcpy(hb + o_off, in->node_offset, 4 * (B + 1));
  if (T) {
    std::memcpy(hb + o_par, in->parent, 4 * T);
    std::memcpy(hb + o_tok, in->token, 4 * T);
  }
  uint8_t* ws = (uint8_t*)workspace;
  uint8_t* din = ws + w.stage_in;
  uint8_t* dou = ws + w.stage_out;
  DevIn di{(int*)(din + o_kv), (int*)(din + o_ctx), (int*)(din + o_root), (int*)(din + o_off),
           (int*)(din + o_par), (int*)(din + o_tok), (uint64_t*)(din + o_ses), (uint32_t*)(din + o_round)};
  DevOut dout{(int*)(dou + q_st), (int*)(dou + q_al), (int*)(dou + q_at), (int*)(dou + q_an), (int*)(dou + q_bo),
              (int*)(dou + q_rt), (float*)(dou + q_rs)};
  uint8_t* ho = hb + in_bytes;
  // H2D of the packed inputs, the verify step, D2H of the packed outputs: one graph replay
  auto step = [&](cudaStream_t gs) -> specedge_status {
    CK(cudaMemcpyAsync(din, hb, in_bytes, cudaMemcpyHostToDevice, gs));
    const specedge_status r = run_verify(m, pool, in, di, dout, ws, ws_bytes, gs, false, in->auto_commit != 0);
    if (r != SPECEDGE_OK) return r;
    CK(cudaMemcpyAsync(ho, dou, out_bytes, cudaMemcpyDeviceToHost, gs));
    return SPECEDGE_OK;
  };
  if (graphs_enabled(m, st))
    s = run_graphed(m, graph_key(in, (const void*)pool, workspace, ws_bytes, (const void*)hb, 2), st, step);
  else
    s = step(st);
  if (s != SPECEDGE_OK) return s;
  CK(cudaStreamSynchronize(st));
  std::memcpy(out->status, ho + q_st, 4 * B);
  std::memcpy(out->accepted_len, ho + q_al, 4 * B);
  std::memcpy(out->bonus, ho + q_bo, 4 * B);
  if (T) {
    std::memcpy(out->accepted_token, ho + q_at, 4 * T);
    std::memcpy(out->accepted_node, ho + q_an, 4 * T);
  }
  if (out->row_target) std::memcpy(out->row_target, ho + q_rt, 4 * R);
  if (out->row_score) std::memcpy(out->row_score, ho + q_rs, 4 * R);
  return SPECEDGE_OK;
}

specedge_status specedge_prefill(specedge_model* m, specedge_kvpool* pool, int32_t h, const int32_t* tokens, int32_t n,
                                 void* workspace, size_t ws_bytes, void* stream) {
  if (!m || !pool || !tokens || n < 1 || h < 0 || h >= pool->max_handles || pool->handle_cap[h] == 0)
    return SPECEDGE_E_INVALID;
  for (int i = 0; i < n; ++i)
    if (tokens[i] < 0 || tokens[i] >= m->cfg.vocab) return SPECEDGE_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  int L = 0;
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(&L, pool->cache_len + h, sizeof(int), cudaMemcpyDeviceToHost));
  if (L + n - 1 > pool->handle_cap[h]) return SPECEDGE_E_INVALID;
  // largest chain chunk whose (1 request, cn + 1 rows) layout fits the caller's workspace
  int max_cn = SPECEDGE_MAX_NODES;
  while (max_cn > 0 && ws_layout(m->cfg, 1, max_cn + 1).total > ws_bytes) --max_cn;
  if (ws_layout(m->cfg, 1, 1).total > ws_bytes) return SPECEDGE_E_WORKSPACE;
  int i = 0;
  while (i < n - 1) {
    const int cn = std::min(max_cn, n - 2 - i);   // chain nodes after the root tokens[i]
    const int B = 1, T = cn, R = T + 1;
    const WsLayout w = ws_layout(m->cfg, B, R);
    if (!workspace || ws_bytes < w.total) return SPECEDGE_E_WORKSPACE;
    // host block: kv, ctx, root, round, session, node_offset[2], parent[T], token[T]
    std::vector<int32_t> blk(8 + 2 * T, 0);
    blk[0] = h;
    blk[1] = L + 1;
    blk[2] = tokens[i];
    blk[3] = 0;
    blk[4] = 0;
    blk[5] = 0;            // session (u64) = 0
    blk[6] = 0;
    blk[7] = T;            // node_offset = {0, T} -> blk[6], blk[7]
    for (int k = 0; k < T; ++k) {
      blk[8 + k] = k - 1;
      blk[8 + T + k] = tokens[i + 1 + k];
    }
    uint8_t* ws = (uint8_t*)workspace;
    uint8_t* din = ws + w.stage_in;
    uint8_t* dou = ws + w.stage_out;
    CK(cudaMemcpyAsync(din, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice, st));
    const int32_t* d32 = (const int32_t*)din;
    specedge_verify_in vin{};
    vin.num_requests = 1;
    vin.total_nodes = T;
    vin.max_nodes = std::max(T, 0);
    vin.max_context_len = std::min(m->cfg.max_position, L + 1);
    vin.mode = SPECEDGE_GREEDY;
    DevIn di{d32 + 0, d32 + 1, d32 + 2, d32 + 6, d32 + 8, d32 + 8 + T, (const uint64_t*)(d32 + 4),
             (const uint32_t*)(d32 + 3)};
    int32_t* o32 = (int32_t*)dou;
    DevOut dout{o32 + 0, o32 + 1, o32 + 4, o32 + 4 + SPECEDGE_MAX_NODES, o32 + 2, nullptr, nullptr};
    specedge_status s = run_verify(m, pool, &vin, di, dout, ws, ws_bytes, st, true, true);
    if (s != SPECEDGE_OK) return s;
    int status = -1;
    CK(cudaMemcpyAsync(&status, o32, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (status != SPECEDGE_REQ_OK) return SPECEDGE_E_INVALID;
    L += T + 1;
    i += T + 1;
  }
  return SPECEDGE_OK;
}

specedge_status specedge_debug_weight_rows(specedge_model* m, int32_t tensor, int32_t layer, int32_t row0, int32_t nrows,
                                           uint16_t* dst) {
  if (!m || !dst || nrows < 0 || row0 < 0) return SPECEDGE_E_INVALID;
  const auto& c = m->cfg;
  const long long H = c.n_heads, KV = c.n_kv, hd = c.head_dim, d = c.d, F = c.ffn;
  if ((tensor >= 2 && tensor <= 8) || tensor == 10 || tensor == 11)
    if (layer < 0 || layer >= c.n_layers) return SPECEDGE_E_INVALID;
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < nrows; ++i) {
    const long long r = row0 + i;
    const bf16* base = nullptr;
    long long cols = d, prow = r, rows = 0;
    switch (tensor) {
      case 1: base = m->embed; rows = c.vocab; break;
      case 2: base = m->layers[layer].wqkv; rows = H * hd; break;
      case 3: base = m->layers[layer].wqkv; rows = KV * hd; prow = H * hd + r; break;
      case 4: base = m->layers[layer].wqkv; rows = KV * hd; prow = (H + KV) * hd + r; break;
      case 5: base = m->layers[layer].wo; rows = d; cols = H * hd; break;
      case 6: base = m->layers[layer].wgu; rows = F; prow = (r / 64) * 128 + r % 64; break;
      case 7: base = m->layers[layer].wgu; rows = F; prow = (r / 64) * 128 + 64 + r % 64; break;
      case 8: base = m->layers[layer].wd; rows = d; cols = F; break;
      case 9: base = m->lm_head; rows = m->vl; break;   // this rank's vocab shard
      case 10: base = m->layers[layer].g_attn; rows = 1; break;
      case 11: base = m->layers[layer].g_mlp; rows = 1; break;
      case 12: base = m->g_final; rows = 1; break;
      default: return SPECEDGE_E_INVALID;
    }
    if (r >= rows) return SPECEDGE_E_INVALID;
    CK(cudaMemcpy(dst + (size_t)i * cols, base + prow * cols, cols * 2, cudaMemcpyDeviceToHost));
  }
  return SPECEDGE_OK;
}

specedge_status specedge_debug_read_kv(specedge_kvpool* p, int32_t h, int32_t layer, int32_t kv_sel, int32_t pos0,
                                       int32_t n, uint16_t* dst) {
  if (!p || !dst || h < 0 || h >= p->max_handles || p->handle_cap[h] == 0 || pos0 < 0 || n < 0 ||
      pos0 + n > p->handle_cap[h] || kv_sel < 0 || kv_sel > 1)
    return SPECEDGE_E_INVALID;
  const auto& c = p->model->cfg;
  if (layer < 0 || layer >= c.n_layers) return SPECEDGE_E_INVALID;
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < n; ++i) {
    const int pos = pos0 + i;
    const int page = p->handle_pages[h][pos / kPage];
    for (int g = 0; g < c.n_kv; ++g) {
      const size_t off = (((((size_t)layer * p->num_pages + page) * 2 + kv_sel) * c.n_kv + g) * kPage + pos % kPage) * c.head_dim;
      CK(cudaMemcpy(dst + ((size_t)i * c.n_kv + g) * c.head_dim, p->pages + off, c.head_dim * 2, cudaMemcpyDeviceToHost));
    }
  }
  return SPECEDGE_OK;
}

specedge_status specedge_debug_read_tree_kv(specedge_model* m, const void* workspace, size_t ws_bytes, int32_t B,
                                            int32_t R, int32_t layer, int32_t kv_sel, int32_t row0, int32_t n,
                                            uint16_t* dst) {
  if (!m || !workspace || !dst || B <= 0 || R < B || layer < 0 || layer >= m->cfg.n_layers || kv_sel < 0 ||
      kv_sel > 1 || row0 < 0 || n < 0 || row0 + n > R)
    return SPECEDGE_E_INVALID;
  const auto& c = m->cfg;
  const WsLayout w = ws_layout(c, B, R);
  if (ws_bytes < w.total) return SPECEDGE_E_WORKSPACE;
  CK(cudaSetDevice(m->device));
  CK(cudaDeviceSynchronize());
  // tree scratch [layer][K|V][kv_head][R][hd] fp16 (R = this batch's rows)
  const uint16_t* base = reinterpret_cast<const uint16_t*>((const uint8_t*)workspace + w.tree_kv);
  for (int g = 0; g < c.n_kv; ++g) {
    const size_t src = ((((size_t)layer * 2 + kv_sel) * c.n_kv + g) * R + row0) * c.head_dim;
    CK(cudaMemcpy2D(dst + (size_t)g * c.head_dim, (size_t)c.n_kv * c.head_dim * 2, base + src, (size_t)c.head_dim * 2,
                    (size_t)c.head_dim * 2, n, cudaMemcpyDeviceToHost));
  }
  return SPECEDGE_OK;
}

specedge_status specedge_debug_gemm(const uint16_t* W, const uint16_t* X, float* out, int32_t M, int32_t R, int32_t K,
                                    void* stream) {
  if (!W || !X || !out || M <= 0 || R <= 0 || K <= 0 || K % 8) return SPECEDGE_E_INVALID;
  CUtensorMap tmW;
  if (!make_tmap_2d(&tmW, W, (uint64_t)M, (uint64_t)K, 128)) return SPECEDGE_E_CUDA;
  GemmArgs g{};
  g.M = M;
  g.R = R;
  g.K = K;
  g.out_f32 = out;
  g.ldo = M;
  CK(gemm_launch(EPI_F32, tmW, X, g, (cudaStream_t)stream, nullptr));
  return SPECEDGE_OK;
}

specedge_status specedge_draft_tree(specedge_model* m, specedge_kvpool* pool, int32_t handle, int32_t context_len,
                                    int32_t root_token, uint64_t session_id, const int32_t* head_tokens,
                                    int32_t head_len, int32_t budget, int32_t depth, int32_t branching,
                                    void* workspace, size_t ws_bytes, void* stream, int32_t* parent_out,
                                    int32_t* token_out, float* logprob_out, int32_t* n_out) {
  if (!m || !pool || pool->model != m || !workspace || !parent_out || !token_out || !logprob_out || !n_out)
    return SPECEDGE_E_INVALID;
  if (budget < 1 || head_len < 0 || head_len + budget > SPECEDGE_MAX_NODES || depth < 1 || branching < 1 ||
      branching > 8 || handle < 0 || handle >= pool->max_handles || context_len < 1 || root_token < 0 ||
      root_token >= m->cfg.vocab || (head_len > 0 && !head_tokens))
    return SPECEDGE_E_INVALID;
  for (int i = 0; i < head_len; ++i)
    if (head_tokens[i] < 0 || head_tokens[i] >= m->cfg.vocab) return SPECEDGE_E_INVALID;
  const int P = head_len;   // proactive expansion: the subtree grows under this fixed chain
  if (m->tp_size != 1) return SPECEDGE_E_UNSUPPORTED;
  const auto& c = m->cfg;
  const int V = c.vocab;
  if (ws_bytes < ws_layout(c, 1, P + budget + 1).total) return SPECEDGE_E_WORKSPACE;
  CK(cudaSetDevice(m->device));
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)workspace;
  std::vector<DraftNode> nodes;
  std::vector<int> frontier{-1};
  for (int pass = 0; pass < depth && !frontier.empty(); ++pass) {
    const int N = P + (int)nodes.size(), R = N + 1;   // tree = head chain ++ subtree
    // the workspace layout of THIS pass's tree (run_verify places its buffers by (B, R)); the
    // staging, logits and top-b buffers are regions a hidden-only forward does not touch
    const WsLayout w = ws_layout(c, 1, R);
    uint8_t* din = ws + w.stage_in;
    uint8_t* dou = ws + w.stage_out;
    int* d_rows = (int*)(ws + w.y);
    int* d_tok = (int*)(ws + w.part_idx);
    float* d_lp = (float*)(ws + w.part_val);
    float* logits = (float*)(ws + w.draft_logits);   // [R][V] fp32
    // inputs: kv, context_len, root_token, round, session (8 B), node_offset[2], parent[N], token[N]
    std::vector<int32_t> h32(5 + 2 + 2 * N + 2);
    h32[0] = handle;
    h32[1] = context_len;
    h32[2] = root_token;
    h32[3] = 0;   // round
    std::memcpy(&h32[4], &session_id, 8);
    h32[6] = 0;
    h32[7] = N;
    for (int i = 0; i < P; ++i) {
      h32[8 + i] = i - 1;
      h32[8 + N + i] = head_tokens[i];
    }
    for (int i = 0; i < N - P; ++i) {
      h32[8 + P + i] = nodes[i].parent < 0 ? P - 1 : P + nodes[i].parent;
      h32[8 + N + P + i] = nodes[i].token;
    }
    CK(cudaMemcpyAsync(din, h32.data(), h32.size() * 4, cudaMemcpyHostToDevice, st));
    int32_t* di32 = (int32_t*)din;
    DevIn di{di32 + 0, di32 + 1, di32 + 2, di32 + 6, di32 + 8, di32 + 8 + N, (const uint64_t*)(di32 + 4),
             (const uint32_t*)(di32 + 3)};
    int32_t* do32 = (int32_t*)dou;
    DevOut dout{do32, do32 + 1, do32 + 2, do32 + 2 + std::max(N, 1), do32 + 2 + 2 * std::max(N, 1), nullptr, nullptr};
    specedge_verify_in vin{};
    vin.num_requests = 1;
    vin.total_nodes = N;
    vin.max_nodes = std::max(N, 1);
    vin.max_context_len = context_len;
    vin.mode = SPECEDGE_GREEDY;
    const specedge_status s = run_verify(m, pool, &vin, di, dout, ws, ws_bytes, st, false, false, true);
    if (s != SPECEDGE_OK) return s;
    GemmArgs g{};
    g.M = V;
    g.R = 2 * R;
    g.pair = 1;
    g.K = c.d;
    g.out_f32 = logits;
    g.ldo = V;
    CK(gemm_launch(EPI_F32, m->tm_lm, ws + w.Hf, g, st, nullptr));
    std::vector<int> rows(frontier.size());
    for (size_t i = 0; i < frontier.size(); ++i) rows[i] = frontier[i] < 0 ? P : P + frontier[i] + 1;   // slot
    CK(cudaMemcpyAsync(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, st));
    CK(topb_launch(logits, V, d_rows, (int)rows.size(), branching, d_tok, d_lp, st));
    std::vector<int> tok(rows.size() * branching);
    std::vector<float> lp(rows.size() * branching);
    int32_t status = -1;
    CK(cudaMemcpyAsync(tok.data(), d_tok, tok.size() * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(lp.data(), d_lp, lp.size() * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&status, do32, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (status != SPECEDGE_REQ_OK) return SPECEDGE_E_INVALID;   // e.g. context_len != cached + 1
    std::vector<int> next;
    const specedge_status ps = draft_prune(nodes, frontier, tok, lp, branching, budget, next);
    if (ps != SPECEDGE_OK) return ps;
    frontier.swap(next);
  }
  *n_out = (int32_t)nodes.size();
  for (size_t i = 0; i < nodes.size(); ++i) {
    parent_out[i] = nodes[i].parent;
    token_out[i] = nodes[i].token;
    logprob_out[i] = nodes[i].logprob;
  }
  return SPECEDGE_OK;
}

specedge_status specedge_debug_last_logits(specedge_model* m, void* workspace, size_t ws_bytes, int32_t B, int32_t R,
                                           float* logits, void* stream) {
  if (!m || !workspace || !logits || B <= 0 || R < B) return SPECEDGE_E_INVALID;
  const WsLayout w = ws_layout(m->cfg, B, R);
  if (ws_bytes < w.total) return SPECEDGE_E_WORKSPACE;
  GemmArgs g{};
  g.M = m->vl;   // this rank's vocab shard
  g.R = 2 * R;
  g.pair = 1;
  g.K = m->cfg.d;
  g.out_f32 = logits;
  g.ldo = m->vl;
  CK(gemm_launch(EPI_F32, m->tm_lm, (uint8_t*)workspace + w.Hf, g, (cudaStream_t)stream, nullptr));
  return SPECEDGE_OK;
}

specedge_status specedge_debug_attention(const uint16_t* q, const uint16_t* k_prefix, const uint16_t* v_prefix,
                                         const uint16_t* k_tree, const uint16_t* v_tree, const uint64_t* anc, int32_t S,
                                         int32_t G, int32_t hd, int32_t L, int32_t n_splits, float* o, void* workspace,
                                         size_t ws_bytes, void* stream) {
  if (!q || !k_tree || !v_tree || !o || S < 1 || S > SPECEDGE_MAX_NODES + 1 || G < 1 || L < 0 ||
      (L > 0 && (!k_prefix || !v_prefix)) || (S > 1 && !anc) || n_splits < 1 || n_splits > kMaxSplits)
    return SPECEDGE_E_INVALID;
  if (!(hd == 16 || hd == 32 || hd == 64 || hd == 128)) return SPECEDGE_E_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const int npages = std::max(1, (L + 63) / 64);
  size_t off = 0;
  auto take = [&](size_t b) { size_t a = off; off = al256(off + b); return a; };
  const size_t o_pool = take((size_t)npages * 2 * 64 * hd * 2), o_bt = take(4 * npages), o_tree = take(2 * 2 * (size_t)S * hd),
               o_req = take(4 * 4), o_anc = take(8 * (size_t)S), o_op = take(4 * (size_t)n_splits * S * G * hd),
               o_m = take(4 * (size_t)n_splits * S * G), o_l = take(4 * (size_t)n_splits * S * G);
  if (!workspace || ws_bytes < off) return SPECEDGE_E_WORKSPACE;
  uint8_t* ws = (uint8_t*)workspace;
  f16* pool = (f16*)(ws + o_pool);
  for (int p = 0; p < (L + 63) / 64; ++p) {
    const int nt = std::min(64, L - p * 64);
    CK(cudaMemcpyAsync(pool + ((size_t)p * 2 + 0) * 64 * hd, k_prefix + (size_t)p * 64 * hd, (size_t)nt * hd * 2,
                       cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(pool + ((size_t)p * 2 + 1) * 64 * hd, v_prefix + (size_t)p * 64 * hd, (size_t)nt * hd * 2,
                       cudaMemcpyDeviceToDevice, st));
  }
  std::vector<int> bt(npages);
  for (int p = 0; p < npages; ++p) bt[p] = p;
  CK(cudaMemcpyAsync(ws + o_bt, bt.data(), 4 * npages, cudaMemcpyHostToDevice, st));
  f16* tree = (f16*)(ws + o_tree);
  CK(cudaMemcpyAsync(tree, k_tree, (size_t)S * hd * 2, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(tree + (size_t)S * hd, v_tree, (size_t)S * hd * 2, cudaMemcpyDeviceToDevice, st));
  const int req[4] = {L, 0, 0, S};   // req_L, req_h, req_row0, req_S
  CK(cudaMemcpyAsync(ws + o_req, req, 16, cudaMemcpyHostToDevice, st));
  const uint64_t zero = 0;
  CK(cudaMemcpyAsync(ws + o_anc, &zero, 8, cudaMemcpyHostToDevice, st));
  if (S > 1) CK(cudaMemcpyAsync(ws + o_anc + 8, anc, 8 * (size_t)(S - 1), cudaMemcpyDeviceToDevice, st));
  AttnArgs a{};
  a.Q = (const f16*)q;
  a.pool = pool;
  a.block_table = (const int*)(ws + o_bt);
  a.max_pages_per_seq = npages;
  a.num_pages = npages;
  a.tree_kv = tree;
  a.R_cap = S;
  a.layer = 0;
  a.H = G;
  a.KV = 1;
  a.G = G;
  a.hd = hd;
  const int* rq = (const int*)(ws + o_req);
  a.req_L = rq;
  a.req_h = rq + 1;
  a.req_row0 = rq + 2;
  a.req_S = rq + 3;
  a.row_anc = (const uint64_t*)(ws + o_anc);
  a.pages_per_split = std::max(1, ((L + 63) / 64 + n_splits - 1) / n_splits);
  a.n_splits = n_splits;
  a.max_rows = S * G;
  a.opart = (float*)(ws + o_op);
  a.mpart = (float*)(ws + o_m);
  a.lpart = (float*)(ws + o_l);
  a.R = S;
  a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)hd));
  if (attention_tc_supported(hd, G)) {
    a.per_req = 1;   // row_req = nullptr: one request
    CK(attention_tc_launch(a, 1, nullptr, o, st, nullptr));
    if (n_splits > 1) CK(attn_combine_launch(a, nullptr, o, st, nullptr));
  } else {
    CK(attention_launch(a, 1, st, nullptr));
    CK(attn_combine_launch(a, nullptr, o, st, nullptr));
  }
  CK(cudaStreamSynchronize(st));
  return SPECEDGE_OK;
}

int32_t specedge_last_launch_count(void) { return g_last_launches; }

specedge_status specedge_set_kernel_timing(int32_t enable) {
  g_timing.on = enable != 0;
  g_timing.mask = enable < 0 ? 0xFFFFFFFFu : (uint32_t)enable;
  return SPECEDGE_OK;
}

specedge_status specedge_kernel_times(float* out_ms, int32_t* out_count, int32_t reset) {
  for (auto& pr : g_timing.pending) {
    cudaEvent_t a = g_timing.pool[pr.second], b = g_timing.pool[pr.second + 1];
    float ms = 0.f;
    if (cudaEventSynchronize(b) != cudaSuccess || cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
      cudaGetLastError();   // do not leave the failure to the next launch check
      g_timing.pending.clear();
      g_timing.used = 0;
      return SPECEDGE_E_CUDA;
    }
    g_timing.ms[pr.first] += ms;
    g_timing.count[pr.first] += 1;
  }
  g_timing.pending.clear();
  g_timing.used = 0;
  for (int k = 0; k < K_NKINDS; ++k) {
    if (out_ms) out_ms[k] = (float)g_timing.ms[k];
    if (out_count) out_count[k] = g_timing.count[k];
    if (reset) {
      g_timing.ms[k] = 0;
      g_timing.count[k] = 0;
    }
  }
  return SPECEDGE_OK;
}

}  // extern "C"
