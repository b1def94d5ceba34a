// Internal declarations shared by the libspecedge translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stddef.h>
#include <atomic>
#include <string>
#include <utility>
#include <vector>

#include "../../include/specedge.h"

namespace se {

// Per-device one-time state.  A process may drive several GPUs (specedge_model_create takes a
// device), and kernel attributes such as the dynamic shared-memory limit are per device: first()
// is true once for each device id it is called under (the current device).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDevices ? 0 : d;
}
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  bool first() {
    const uint64_t bit = 1ull << current_device();
    return !(done.fetch_or(bit) & bit);
  }
};
// SM count of the current device (cached per device id)
inline int device_sms() {
  static std::atomic<int> n[kMaxDevices];
  const int d = current_device();
  int v = n[d].load();
  if (v <= 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    if (v <= 0) v = 148;
    n[d].store(v);
  }
  return v;
}

// Launch with programmatic stream serialisation (kernels call pdl_begin() before any global
// access; SPECEDGE_PDL=0 turns it off).
bool pdl_enabled();
// Every kernel of the step asks for the max-shared-memory carveout (the GEMMs and the attention
// need it), so consecutive kernels never change the SM's L1 / shared split (SPECEDGE_CARVEOUT=0:
// driver default for the small kernels).  Once per (kernel, device).
bool carveout_first(const void* kern);
void carveout_skip(const void* kern);   // leave this kernel at the driver default
int carveout_mode();                    // SPECEDGE_CARVEOUT: 1 (default) all kernels, 2 all but RMSNorm, 0 none
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  if (carveout_first(reinterpret_cast<const void*>(kern)))
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

using bf16 = __nv_bfloat16;
using f16 = __half;   // attention operands q, k, v and the KV cache

// ---------------------------------------------------------------------------------------------
// GEMM (tcgen05, swap-AB: weights are the MMA's M side, activation rows its N side)
// ---------------------------------------------------------------------------------------------
enum GemmMode : int {
  EPI_F32 = 0,     // out_f32[split][row][m] = partial acc (a4 QKV, a6 O, a8 down; logits capture)
  EPI_SWIGLU = 3,  // M[row][f] = bf16(silu(gate) * up)            (a7)
  EPI_ARGMAX = 4,  // per (row, 128-vocab tile) max / Gumbel-max   (a9)
  EPI_PQ1 = 5,     // NEXT-F2 pass 1: EPI_ARGMAX (Gumbel-max) + per-tile (max, sum exp) of l/T
  EPI_PQ2 = 6,     // NEXT-F2 pass 2: per-tile Gumbel-max of log max(0, p - q) + p(child token)
  EPI_QKV = 7,     // a4 with RoPE fused (head_dim 128, unsplit): q -> Q fp16, k/v -> tree K/V fp16
};

constexpr int kMaxFusedTp = 8;   // NEXT-F4: ranks of the fused GEMM -> reduce-scatter (a box's 8 GPUs)
struct RmsSrc {                  // NEXT-F4: per-partial base pointers for k_rmsnorm (p[0] == null: unused)
  const float* mc;               // NVLS: multicast address of this rank's rows (the rank sum is loaded)
  const float* p[kMaxFusedTp];
  bf16* outp[kMaxFusedTp];       // NEXT-F4 all-gather: the normalised row also goes to every rank
  int nout;                      // (split == 0 only); 0: unused
};

struct GemmArgs {
  int M, R, K;            // weight rows (features), activation rows, reduction length
  int bn_override;        // activation-row tile (multiple of 16, <= 256); 0: gemm_pick_bn(R)
  int x_stride;           // activation row stride in elements (0: K); the hi-only LM head reads
                          // the even (hi) rows of the interleaved hi/lo final hidden
  int BN, n_tiles_n, n_tiles_m, num_kb, stages, tmem_cols;
  int ntm128;             // 128-feature tiles (stride of the ARGMAX partials)
  int pair;               // EPI_F32/EPI_ARGMAX: rows (2r, 2r+1) are hi/lo bf16 parts of row r
  int nc;                 // CTA-pair kernel: pairs per cluster sharing one weight tile (TMA multicast)
  int n_groups;           // CTA-pair kernel: ceil(n_tiles_n / nc) (mcx: ceil(256-feature pairs / nc))
  int mcx;                // CTA-pair kernel: the nc pairs of a cluster share the ACTIVATION tile (pair
                          // qp takes weight tile group * nc + qp, pair 0 multicasts X) instead of the
                          // weight tile
  int splits, kb_per_split, max_splits;   // K-split (EPI_F32): slice sk at out_f32 + sk*split_stride
  int unsplit_if_full;    // EPI_F32: no K-split when the tiles already fill >= 90 % of one wave
  // CTA-pair kernel, last-wave K split (EPI_SWIGLU): tiles [0, n_full) run whole (or in `splits`
  // K-slices); each tile t >= n_full runs as tail_split K-parts of kb_tail k-blocks whose fp32
  // accumulators go to tail_buf, and the last part of (tile, pair, half) to finish (counter in
  // tile_cnt) sums them in part order and runs the epilogue (set by gemm_launch; tail_buf /
  // tail_cap / tile_cnt from the caller, nullptr: no tail split)
  int n_full, tail_split, kb_tail;
  float* tail_buf;
  size_t tail_cap;        // bytes
  size_t split_stride;
  // EPI_F32 / EPI_RESID (fp32 residual stream)
  float* out_f32;
  int ldo;
  // EPI_F32 fused residual add (a6 / a8; CTA-pair kernel): resid[row][f] += the unit's K-split
  // partials.  splits == 1: the epilogue adds its accumulator straight into resid; splits > 1:
  // every split stores its partial, and the last of the tile's splits to finish (a per-(tile,
  // half) counter in tile_cnt, zero between launches) computes ((X + Y0) + Y1) + ... in split order
  // (the same order as k_rmsnorm's sum: deterministic) and stores it into resid.
  float* resid;
  int* tile_cnt;
  // EPI_F32 with push (NEXT-F4): each 32-row chunk is staged in shared memory and row r is sent
  // with a bulk async copy to rank o = r / rows_per_rank, slot [tp_src] of its receive buffer:
  // peer_out[o] + tp_src * slot_stride + (r - o * rows_per_rank) * ldo
  int push, tp_src, rows_per_rank;
  size_t slot_stride;
  float* peer_out[kMaxFusedTp];
  // EPI_SWIGLU / EPI_QKV(q part)
  bf16* out_bf16;
  int ld_out;
  // EPI_QKV
  bf16* tree_kv;          // [layers][2][KV][R_cap][hd]
  int R_cap, layer, n_heads, n_kv, head_dim;
  const int* row_pos;
  const float* rope_cos;  // [max_pos][hd/2]
  const float* rope_sin;
  // EPI_ARGMAX
  float* part_val;        // [R][n_tiles_m]
  int* part_idx;
  int top2;               // also store the tile's second-best (score, id) and third score: hi-only LM head
  float* part_val2;
  int* part_idx2;
  float* part_val3;
  int vocab, sample;      // vocab: rows of this (vocab-shard) LM head
  int vocab_off;          // global id of local row 0 (tensor parallel vocab shard)
  float inv_t;
  uint32_t seed_lo, seed_hi;
  const int* row_req;
  const int* row_slot;
  const uint32_t* req_round;
  const uint64_t* req_session;
  // EPI_PQ1 / EPI_PQ2 (dense-q speculative sampling, SAMPLE_PQ_DENSE)
  float* part_m;          // [R][n_tiles_m] tile max of l/T          (PQ1)
  float* part_s;          // [R][n_tiles_m] tile sum exp(l/T - max)  (PQ1)
  const float* lse;       // [R] log sum exp(l/T)                     (PQ2)
  const int* row_qnode;   // [R] node drawn at this slot (its q row), -1 for the last slot
  const int* node_token;  // [total_nodes]
  const float* draft_q;   // [total_nodes][vocab_q] fp32
  int vocab_q;            // row stride of draft_q (= V)
  float* pchild;          // [R] p(child token) at this slot          (PQ2)
};

// Build a 2D bf16 tensor map [rows][cols] (cols contiguous), box {64, box_rows}, 128B swizzle.
// row_stride: elements between rows (0: cols, i.e. contiguous rows)
bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                  uint64_t row_stride = 0);
int gemm_pick_bn(int R);
bool gemm_qkv_fused_ok(int M, int R);
int gemm_splits_last();   // K-splits chosen by the last gemm_launch on this thread
void gemm_force_single(bool on);   // tests/probes: disable the CTA-pair kernel
cudaError_t gemm_launch(int mode, const CUtensorMap& tmW, const void* X, GemmArgs a,
                        cudaStream_t st, int* launches);

// ---------------------------------------------------------------------------------------------
// Attention (tree-masked, paged, split-KV)
// ---------------------------------------------------------------------------------------------
struct AttnArgs {
  const f16* Q;               // [R][H*hd]
  const f16* pool;            // [layers][num_pages][2][KV][64][hd]
  const int* block_table;     // [max_handles][max_pages_per_seq]
  int max_pages_per_seq, num_pages;
  const f16* tree_kv;         // [layers][2][KV][R_cap][hd]
  int R_cap, layer, H, KV, G, hd;
  const int* req_L;
  const int* req_h;
  const int* req_row0;
  const int* req_S;
  const uint64_t* row_anc;
  int n_splits, pages_per_split, max_rows;   // max_rows = max_S * G
  float* opart;               // [n_splits][R][H][hd]
  float* mpart;               // [n_splits][R][H]   (log2 domain)
  float* lpart;
  int R;
  float scale_log2;
  // per_req = 1 (tcgen05 path): request r has its own chunk count max(1, ceil(pages_r /
  // pages_per_split)) <= n_splits, the tree keys go to its last chunk, and a request with one
  // chunk is written final by the attention kernel (the combine skips its rows, via row_req;
  // row_req == nullptr means every row belongs to request 0).  per_req = 0: every request has
  // n_splits splits, the tree in the last one (the mma.sync kernel).
  // per_req = 2 (tcgen05, balanced): a persistent grid of grid_ctas CTAs splits the concatenated
  // (r, g) sub-tile sequences evenly (attention_tc.cu); chunks per (r, g) <= n_splits.
  int per_req;
  const int* row_req;
  int B, grid_ctas;
  int* nch_tab;               // per_req = 2: [B][KV] chunk counts, written by the attention kernel
  int* merge_cnt;             // per_req = 2 with merge_cnt: [B][KV] finished-chunk counters (zero
                              // between launches); the last CTA per (r, g) merges (null: combine kernel)
};
cudaError_t attention_launch(const AttnArgs& a, int B, cudaStream_t st, int* launches);
cudaError_t attn_combine_launch(const AttnArgs& a, bf16* O, float* O_f32, cudaStream_t st,
                                int* launches);
int attn_pick_splits(int B, int KV, int max_pages);
int attn_pick_chunk_tc(int B, int KV, int max_pages);   // pages per chunk (per_req = 1)
// tcgen05 attention (head_dim 64 / 128); with n_splits == 1 it writes the normalised output
// directly (bf16 O and/or fp32 O_f32), otherwise (o, m, l) partials for attn_combine_launch.
bool attention_tc_supported(int hd, int G);
cudaError_t attention_tc_launch(const AttnArgs& a, int B, bf16* O, float* O_f32, cudaStream_t st, int* launches);

// ---------------------------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------------------------
struct PrepArgs {
  int B, V, max_nodes, max_context_len, max_handles, force_chain, max_position;
  const int* kv;
  const int* context_len;
  const int* root_token;
  const int* node_offset;
  const int* parent;
  const int* token;
  const int* cache_len;
  const int* capacity;
  // outputs
  int* status;
  int* req_L;
  int* req_h;
  int* req_row0;
  int* req_S;
  int* row_tok;
  int* row_pos;
  int* row_req;
  int* row_slot;
  uint64_t* row_anc;
};
cudaError_t prep_launch(const PrepArgs& p, cudaStream_t st, int* launches);
cudaError_t embed_launch(const bf16* E, const int* row_tok, float* X, int R, int d, cudaStream_t st,
                         int* launches);
// x = X + sum_s Y[s] (s < nY, fixed order; X updated in place), out = bf16(rmsnorm(x) * g);
// split = 1 writes out as hi/lo bf16 row pairs (LM-head input).
cudaError_t rmsnorm_launch(float* X, const float* Y, int nY, size_t y_stride, const bf16* g, bf16* out,
                           int R, int d, float eps, cudaStream_t st, int* launches, int split = 0,
                           const RmsSrc* ys = nullptr);
// Q / tree K/V from the QKV GEMM's fp32 split partials: sum splits, RoPE(q, k) at row_pos,
// bf16 round, scatter
struct RopeArgs {
  const float* Y;
  int nY;
  size_t y_stride;
  int R, H, KV, hd, layer, R_cap;
  const int* row_pos;
  const float* rope_cos;
  const float* rope_sin;
  f16* Q;
  f16* tree_kv;
};
cudaError_t qkv_rope_launch(const RopeArgs& r, cudaStream_t st, int* launches);
cudaError_t lm_reduce_launch(const float* pv, const int* pi, int R, int ntiles, int* y, float* score,
                             int* row_target, float* row_score, cudaStream_t st, int* launches);
// a9 second stage of the hi-only LM head (k_lm_refine): the GEMM scores every vocab id with the
// hi part of the final hidden only; per (row, tile) it keeps the best two (value, id) and the third
// best value.  |lo . W_v| <= ||lo||_2 max_v ||W_v||_2 (Cauchy-Schwarz), so the true argmax of
// (hi + lo) . W lies among the ids whose hi score is within W_r = 2 (||lo|| + rho) wmax scale of the
// best hi score (rho: fp32 accumulation error bound); every such candidate (a tile's best and
// second, or all 128 ids of a tile whose third best also falls in the window) is rescored exactly
// with (hi + lo) . W_v on the CUDA cores, and the argmax of the rescored set (ties -> lowest id) is
// the row's target.
struct RefineArgs {
  int R, ntiles, d, vocab, vocab_off, sample;
  float inv_t, wmax;
  const float* part_val;    // [R][ntiles]
  const int* part_idx;      // [R][ntiles] global ids
  const float* part_val2;   // [R][ntiles]
  const int* part_idx2;     // [R][ntiles]
  const float* part_val3;   // [R][ntiles]
  const bf16* hf;           // [2R][d]: hi row 2r, lo row 2r+1
  const bf16* w;            // LM head shard [vocab][d]
  uint32_t seed_lo, seed_hi;
  const int* row_req;
  const int* row_slot;
  const uint32_t* req_round;
  const uint64_t* req_session;
  int* y;
  float* score;
  int* row_target;          // nullable
  float* row_score;         // nullable
};
cudaError_t lm_refine_launch(const RefineArgs& a, cudaStream_t st, int* launches);
// max over rows of ||W_v||_2 (fp32) of a [rows][d] bf16 matrix into *out (device float, >= 0)
cudaError_t row_norm_max_launch(const bf16* w, int rows, int d, float* out, cudaStream_t st);
struct WalkArgs {
  int B, force_chain;
  const int* status;
  const int* node_offset;
  const int* parent;
  const int* token;
  const int* y;
  int* accepted_len;
  int* accepted_token;
  int* accepted_node;
  int* bonus;
};
cudaError_t walk_launch(const WalkArgs& w, cudaStream_t st, int* launches);
// NEXT-F2 (SAMPLE_PQ_DENSE): log-sum-exp from the PQ1 tile partials, the q row of every slot, and
// the Leviathan walk over a sampled chain (kernels_small.cu)
struct PqArgs {
  int B, R, ntiles, V;
  int* status;
  const int* node_offset;
  const int* parent;
  const int* token;
  const float* draft_q;        // [total_nodes][V]
  const int* row_req;
  const int* row_slot;
  const float* part_m;         // [R][ntiles]
  const float* part_s;
  float* lse;                  // [R]
  int* row_qnode;              // [R]
  const float* pchild;         // [R]
  const int* y;                // [R] Gumbel-max of l/T (leaf bonus)
  const int* resid_y;          // [R] Gumbel-max of log max(0, p - q) (rejection bonus)
  uint32_t seed_lo, seed_hi;
  const uint32_t* req_round;
  const uint64_t* req_session;
  int* accepted_len;
  int* accepted_token;
  int* accepted_node;
  int* bonus;
};
cudaError_t pq_lse_launch(const PqArgs& a, cudaStream_t st, int* launches);
// NEXT-F3 draft-tree builder (draft.cu)
struct DraftNode {
  int parent, token, depth;
  float logprob;
  double cum;
};
cudaError_t topb_launch(const float* logits, int V, const int* rows, int nrows, int b, int* out_tok, float* out_lp,
                        cudaStream_t st);
specedge_status draft_prune(std::vector<DraftNode>& nodes, const std::vector<int>& frontier,
                            const std::vector<int>& tok, const std::vector<float>& lp, int branching, int budget,
                            std::vector<int>& next_frontier);
cudaError_t pq_walk_launch(const PqArgs& a, cudaStream_t st, int* launches);
struct CommitArgs {
  int B, layers, KV, hd, R_cap, num_pages, max_pages_per_seq;
  int* status;
  const int* req_L;
  const int* req_h;
  const int* req_row0;
  const int* node_offset;
  const int* accepted_len;
  const int* accepted_node;
  const f16* tree_kv;
  f16* pool;
  const int* block_table;
  int* cache_len;
};
cudaError_t commit_launch(const CommitArgs& c, cudaStream_t st, int* launches);

// weights (K12) and synthetic KV (K13)
enum InitLayout : int { INIT_PLAIN = 0, INIT_QKV = 1, INIT_GATEUP = 2 };
struct InitArgs {
  bf16* dst;
  long long rows, cols;       // physical rows/cols
  int layout;
  int tid0, tid1, tid2;       // tensor ids (plain: tid0; qkv: q,k,v; gateup: g,u)
  int layer;
  long long rows0, rows1;     // qkv: q rows, k rows; gateup: F
  float scale0, scale1, scale2;
  int gain;                   // 1: bf16(i24*2^-25 + 1)
  uint32_t k0, k1;
  // tensor-parallel shards: element (prow, col) of the local tensor is element
  // (off[part] + lrow, col0 + col) of the global [*, gcols] matrix of its part
  long long off0, off1, off2, col0, gcols;
};
cudaError_t init_weights_launch(const InitArgs& a, cudaStream_t st);
constexpr int kSetLenBatch = 128;
struct SetLenArgs {
  int n;
  int handle[kSetLenBatch];
  int len[kSetLenBatch];
};
cudaError_t set_len_launch(int* cache_len, const SetLenArgs& a, cudaStream_t st);

// tensor parallelism (tp.cu): NCCL resolved at run time
constexpr int kMaxTp = 16;
bool tp_available();
// NEXT-F4 fused GEMM -> reduce-scatter over NVLink peer memory (tp.cu)
int tp_fused_enable(specedge_model* m, int max_rows, cudaStream_t st);
cudaError_t tp_fused_signal(specedge_model* m, cudaStream_t st, int* launches);
cudaError_t tp_fused_wait(specedge_model* m, cudaStream_t st, int* launches);
void tp_fused_close(specedge_model* m);
int tp_nvls_enable(specedge_model* m, int max_rows, cudaStream_t st);
void tp_nvls_close(specedge_model* m);
int tp_unique_id(uint8_t* out128);
int tp_comm_init(void** comm, const uint8_t* id128, int rank, int size);
void tp_comm_destroy(void* comm);
cudaError_t tp_allreduce_f32(float* buf, size_t n, void* comm, cudaStream_t st);
cudaError_t tp_reduce_scatter_f32(float* buf, size_t per_rank, int rank, void* comm, cudaStream_t st);
cudaError_t tp_all_gather_bf16(bf16* buf, size_t per_rank, int rank, void* comm, cudaStream_t st);
cudaError_t tp_argmax_gather(int* y, float* score, int R, float* gather, int tp, void* comm, int* row_target,
                             float* row_score, cudaStream_t st, int* launches);
cudaError_t kv_fill_launch(f16* pool, const int* block_row, int layers, int num_pages, int KV,
                           int hd, int n_tokens, uint32_t k0, uint32_t k1, uint32_t stream_id, int kv_head0,
                           cudaStream_t st);

}  // namespace se

// ---------------------------------------------------------------------------------------------
// opaque handle definitions
// ---------------------------------------------------------------------------------------------
struct specedge_model {
  specedge_model_config cfg;    // rank-local shapes: n_heads, n_kv, ffn are this rank's shares
  specedge_model_config gcfg;   // global model
  int device;
  int tp_rank = 0, tp_size = 1;
  int v0 = 0, vl = 0;           // LM-head vocab shard [v0, v0 + vl)
  void* nccl = nullptr;         // ncclComm_t when tp_size > 1
  float* tp_gather = nullptr;   // [tp_size][R_max][2] (score, id) all-gather buffer
  int tp_gather_rows = 0;
  // NEXT-F4 (tp.cu): this rank's row-parallel GEMM output [R_max][d] fp32 + flag words [tp],
  // the peers' mappings of theirs, the epoch of the last signalled collective
  int tp_fused_rows = 0;                 // capacity (rows); 0 = fused path off
  // NEXT-F4 NVLS variant (SPECEDGE_TP_F4=nvls): one multicast object over all ranks' [2][R_max][d]
  // fp32 partial buffers; the row-parallel GEMM stores into its own unicast mapping, the owner's
  // RMSNorm reads the rank sum with multimem.ld_reduce through the multicast mapping
  bool tp_nvls = false;
  float* tp_nvls_uc = nullptr;           // this rank's physical buffer (unicast VA)
  float* tp_nvls_mc = nullptr;           // the multicast VA (reads reduce over every rank)
  size_t tp_nvls_bytes = 0, tp_nvls_buf = 0;   // mapped size, floats per half
  unsigned long long tp_nvls_mem = 0, tp_nvls_mch = 0;   // CUmemGenericAllocationHandle x2
  bool tp_nvls_bound = false;
  float* tp_recv = nullptr;              // pull: [R_max][d]; push: [2][tp][ceil(R_max/tp)][d]
  size_t tp_fused_slot = 0;              // push: floats per [src] slot
  se::bf16* tp_hn = nullptr;             // all-gathered normalised rows [R_max][d] (this rank's copy)
  se::bf16* tp_peer_hn[se::kMaxFusedTp] = {};
  int tp_fused_buf = 0;                  // push: receive buffer of the next collective
  float* tp_peer_recv[se::kMaxFusedTp] = {};
  unsigned long long* tp_flags = nullptr;
  unsigned long long** tp_peer_flags_dev = nullptr;
  unsigned long long tp_epoch = 0;
  std::vector<void*> tp_ipc_opened;
  se::bf16* embed = nullptr;
  se::bf16* lm_head = nullptr;
  float lm_wmax = 0.f;          // max_v ||W_v||_2 of this rank's LM-head rows (k_lm_refine window)
  se::bf16* g_final = nullptr;
  struct Layer {
    se::bf16 *wqkv, *wo, *wgu, *wd, *g_attn, *g_mlp;
    CUtensorMap tm_qkv, tm_o, tm_gu, tm_d;
  };
  std::vector<Layer> layers;
  CUtensorMap tm_lm;
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  std::vector<void*> allocs;
  void* pinned = nullptr;       // staging for specedge_verify_batch_host
  size_t pinned_bytes = 0;
  // CUDA-graph cache of whole verify steps (runtime.cu): one instantiated graph per distinct
  // (scalars, buffers) signature, replayed on a model-owned stream ordered after the caller's
  struct Graph {
    std::string key;
    cudaGraphExec_t exec;
  };
  std::vector<Graph> graphs;        // up to 32 instantiated signatures, most recent first
  std::vector<std::string> graph_seen;   // signatures used once (captured on their second use)
  int64_t graph_stats[3] = {0, 0, 0};    // replays, captures, plain (uncaptured) runs
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
};

struct specedge_kvpool {
  specedge_model* model;
  int num_pages, max_handles, max_pages_per_seq;
  se::f16* pages = nullptr;     // [layers][num_pages][2][KV][64][hd] fp16
  int* block_table = nullptr;   // device [max_handles][max_pages_per_seq]
  int* cache_len = nullptr;     // device [max_handles]
  int* capacity = nullptr;      // device [max_handles] (0 = free handle)
  std::vector<int> free_pages;
  std::vector<std::vector<int>> handle_pages;
  std::vector<int> handle_cap;  // host mirror, 0 = free
};
