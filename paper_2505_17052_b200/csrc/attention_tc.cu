// Tree-masked paged split-KV attention on tcgen05 ("custom attention
// masking for each token sequence in the batch ... without cross-sequence interference").
//
// One CTA per (request r, kv head g, split sp).  Query rows of the item are the request's S slots
// x the G query heads sharing kv head g (row = s*G + j); they are cut into M-tiles of
// G*floor(128/G) rows, processed two at a time.  Keys stream in tiles of 128 (two 64-token pages
// of the paged cache, then — in the last split — one tile of the S tree slots from the tree K/V
// scratch, masked by the uint64 ancestor-or-self bitmask).
//
//   warp 0      TMA producer: Q tiles (3-D map over Q[R][H][hd]), K/V tiles (2-D maps over the
//               page pool and the tree scratch), 2-stage ring
//   warp 1      TMEM allocator + MMA issuer (one elected thread):
//                 S_m  = Q_m K^T          kind::f16, A,B from smem (K-major), D fp32 in TMEM
//                 O_m += P_m V            A = P (fp16) from TMEM, B = V from smem (MN-major, 128B
//                                         swizzle); q, k, v are fp16 (DESIGN.md R-precision)
//   warps 2-5   softmax + epilogue of M-tile 0 (one thread = one query row: row max and sum
//   warps 6-9   softmax + epilogue of M-tile 1   need no cross-thread reduction)
//
// Softmax in the log2 domain with a lazily updated running max (O is rescaled only when the max
// grows by more than 8, exact because l uses the same max).  P enters PV as fp16 (11-bit
// significand: ~2e-4 relative error; bf16 P would give ~1.5e-3, SURVEY amb. A12).  The 128 scores
// of a row stay in registers between the max and the exp pass.  TMEM: per M-tile 128 columns S
// (P aliases its first 64) + HD columns O.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace se {

namespace {

constexpr int kWarps = 10;      // producer, MMA, 8 softmax/epilogue warps (2 per TMEM lane quarter)
constexpr int kThreads = kWarps * 32;
constexpr int kStages = 3;      // K/V ring depth (128-key tiles)

// UMMA smem descriptor for an MN-major operand, 128B swizzle: SBO = 1024 B between 8-row
// (K) groups, LBO = stride between 64-element MN atoms.
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::f16 instruction descriptor, A/B fp16 (format 0), D fp32, M x N; bmn: B MN-major (bit 16)
__device__ __forceinline__ uint32_t idesc_f16(int M, int N, bool bmn) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24) | (bmn ? (1u << 16) : 0u);
}

__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack2_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct TcArgs {
  AttnArgs a;
  bf16* O;          // final output when n_splits == 1 (normalised, bf16) else nullptr
  float* O_f32;     // optional fp32 normalised output (debug) when n_splits == 1
  int slots_per_mt; // floor(128 / G)
  unsigned long long* trace;   // debug: per-phase clock64 stamps of CTA 0 (nullptr in production)
};

#define TRACE(slot)                                                                   \
  do {                                                                                \
    if (ta.trace && blockIdx.x == 0 && blockIdx.y == 0) ta.trace[(slot)] = clock64(); \
  } while (0)

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmPool,
              const __grid_constant__ CUtensorMap tmTree, const __grid_constant__ TcArgs ta) {
  constexpr int KB = HD / 64;                  // 64-element hd blocks
  constexpr uint32_t QT_BYTES = 128 * HD * 2;  // one M-tile of Q
  constexpr uint32_t KT_BYTES = 128 * HD * 2;  // one 128-key tile of K (or V)
  constexpr int NST = kStages;
  const AttnArgs& a = ta.a;
  // Q + 3 K/V stages take 224 KB of the 227 KB: the 1024-B alignment SW128 needs comes from the
  // dynamic-smem base itself (no static smem in this kernel); checked below.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem;                              // [KB][128 rows][128 B]
  uint8_t* sK = sQ + QT_BYTES;                     // [NST][KB][128 keys][128 B]
  uint8_t* sV = sK + NST * KT_BYTES;               // [NST][KB][128 keys][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + NST * KT_BYTES);
  uint64_t* q_full = bars;              // [1]
  uint64_t* q_empty = bars + 1;         // [1]
  uint64_t* kv_full = bars + 2;         // [NST]
  uint64_t* kv_empty = kv_full + NST;   // [NST]
  uint64_t* s_full = kv_empty + NST;    // [2 streams][2 buffers]  S_h(t) in buffer t&1
  uint64_t* p_full = s_full + 4;        // [2][2]
  uint64_t* pv_done = p_full + 4;       // [2][2]  PV_h(t) complete
  uint64_t* o_full = pv_done + 4;       // [1]
  uint64_t* o_empty = o_full + 1;       // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);
  uint64_t* s_anc = reinterpret_cast<uint64_t*>(o_empty + 3);  // [66]
  float* s_ml = reinterpret_cast<float*>(s_anc + 66);          // [2 streams][m,l][128 rows]

  const int r = blockIdx.x / a.KV, g = blockIdx.x % a.KV, sp = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
  const int S = min(a.req_S[r], a.max_rows / G);
  const int L = a.req_L[r];
  const int row0 = a.req_row0[r];
  const int h = a.req_h[r];
  const int spm = ta.slots_per_mt;
  const int n_mt = (S + spm - 1) / spm;        // passes: one 128-row M-tile each
  const int npages = (L + 63) / 64;
  const int p_begin = sp * a.pages_per_split;
  const int p_end = min(npages, p_begin + a.pages_per_split);
  const int n_prefix_tiles = max(0, (p_end - p_begin + 1) / 2);
  const bool has_tree = sp == a.n_splits - 1;
  const int ntiles = n_prefix_tiles + (has_tree ? 1 : 0);
  // KV tile visited at step t of pass mt: odd passes walk backwards (tree tile first), so they
  // start on the tiles the previous pass left in L2
  auto tile_of = [&](int mt, int t) {
    if (!(mt & 1)) return t;
    if (has_tree && t == 0) return n_prefix_tiles;
    return n_prefix_tiles - 1 - (t - (has_tree ? 1 : 0));
  };

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    tma_prefetch(&tmQ);
    tma_prefetch(&tmPool);
    tma_prefetch(&tmTree);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 256);
    fence_barrier_init();
  }
  for (int s = threadIdx.x; s < S && s <= kMaxNodes; s += blockDim.x) s_anc[s] = a.row_anc[row0 + s];
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // TMEM columns: stream h owns S buffers [128h, 128h+64) and [128h+64, 128h+128) and the O
  // accumulator [256+128h, 256+128h+HD)
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRACE(322);

  if (warp == 0) {
    // ------------------------------------------------------------------------- TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const int* pages = a.block_table + (size_t)h * a.max_pages_per_seq + p_begin;
      const int np = p_end - p_begin;
      for (int mt = 0; mt < n_mt; ++mt) {
        // page ids of the next prefix tile, loaded one tile ahead of their use
        int pg0 = np > 0 ? __ldg(pages) : 0, pg1 = np > 1 ? __ldg(pages + 1) : pg0;
        mbar_wait(q_empty, (mt & 1) ^ 1);
        mbar_expect_tx(q_full, (uint32_t)(64 * G * spm * 2) * KB);
        for (int kb = 0; kb < KB; ++kb) tma_load_3d(sQ + kb * 128 * 128, &tmQ, q_full, kb * 64, g * G, row0 + mt * spm);
        const bool rev = mt & 1;   // odd passes walk the tiles backwards (L2 reuse of the last tiles)
        if (rev && n_prefix_tiles > 0) {
          const int tl = n_prefix_tiles - 1;
          pg0 = __ldg(pages + 2 * tl);
          pg1 = 2 * tl + 1 < np ? __ldg(pages + 2 * tl + 1) : pg0;
        }
        for (int t = 0; t < ntiles; ++t) {
          mbar_wait(&kv_empty[stage], phase ^ 1);
          mbar_expect_tx(&kv_full[stage], 2 * KT_BYTES);
          uint8_t* dk = sK + stage * KT_BYTES;
          uint8_t* dv = sV + stage * KT_BYTES;
          const int tt = tile_of(mt, t);
          if (tt < n_prefix_tiles) {
            const int cur0 = pg0, cur1 = pg1;
            const int tn = rev ? tt - 1 : tt + 1;   // next prefix tile
            if (tn >= 0 && tn < n_prefix_tiles) {
              pg0 = __ldg(pages + 2 * tn);
              pg1 = 2 * tn + 1 < np ? __ldg(pages + 2 * tn + 1) : pg0;
            }
            for (int hf = 0; hf < 2; ++hf) {
              const int page = hf ? cur1 : cur0;   // odd tail: page 2t reloaded, masked later
              const int rk = (((a.layer * a.num_pages + page) * 2 + 0) * a.KV + g) * 64;
              const int rv = rk + a.KV * 64;
              for (int kb = 0; kb < KB; ++kb) {
                tma_load_2d(dk + kb * 128 * 128 + hf * 64 * 128, &tmPool, &kv_full[stage], kb * 64, rk);
                tma_load_2d(dv + kb * 128 * 128 + hf * 64 * 128, &tmPool, &kv_full[stage], kb * 64, rv);
              }
            }
          } else {
            const int rk = ((a.layer * 2 + 0) * a.KV + g) * a.R_cap + row0;
            const int rv = ((a.layer * 2 + 1) * a.KV + g) * a.R_cap + row0;
            for (int hf = 0; hf < 2; ++hf)
              for (int kb = 0; kb < KB; ++kb) {
                tma_load_2d(dk + kb * 128 * 128 + hf * 64 * 128, &tmTree, &kv_full[stage], kb * 64, rk + 64 * hf);
                tma_load_2d(dv + kb * 128 * 128 + hf * 64 * 128, &tmTree, &kv_full[stage], kb * 64, rv + 64 * hf);
              }
          }
          if (mt == 0) TRACE(t);
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------------- MMA issuer
    if (elect_one()) {
      const uint32_t id_qk = idesc_f16(128, 64, false);
      const uint32_t id_pv = idesc_f16(128, HD, true);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t sfill = 0;        // S tiles filled so far per stream (all passes): buffer = sfill & 1
      uint32_t pcons = 0;        // P tiles consumed so far per stream
      // S_hs = Q K_hs^T for the 64 keys [64hs, 64hs+64) of the tile in stage `st`
      auto issue_qk = [&](int st) {
        const uint32_t qaddr = smem_u32(sQ);
        const uint32_t kaddr = smem_u32(sK + st * KT_BYTES);
#pragma unroll
        for (int hs = 0; hs < 2; ++hs) {
          const uint32_t s_tm = tmem + hs * 128 + (sfill & 1) * 64;
#pragma unroll
          for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16(s_tm, umma_desc_sw128(qaddr + kb * 16384 + k * 32),
                         umma_desc_sw128(kaddr + kb * 16384 + hs * 8192 + k * 32), id_qk, (kb | k) != 0);
          tc_commit(&s_full[hs * 2 + (sfill & 1)]);
        }
        ++sfill;
      };
      for (int mt = 0; mt < n_mt; ++mt) {
        mbar_wait(q_full, mt & 1);
        mbar_wait(o_empty, (mt & 1) ^ 1);   // previous pass's O has been drained
        tc_fence_after();
        if (ntiles > 0) {
          mbar_wait(&kv_full[stage], phase);
          tc_fence_after();
          issue_qk(stage);
        }
        for (int t = 0; t < ntiles; ++t) {
          int nst = stage + 1;
          uint32_t nph = phase;
          if (nst == NST) { nst = 0; nph ^= 1; }
          // S(t+1) into the other S buffers while the softmax works on S(t).  In-order tcgen05
          // execution: S(t+1) overwrites P(t-1) only after PV(t-1), issued before it, has read it.
          if (t + 1 < ntiles) {
            mbar_wait(&kv_full[nst], nph);
            tc_fence_after();
            issue_qk(nst);
          }
          const uint32_t b = pcons & 1;
          const uint32_t vaddr = smem_u32(sV + stage * KT_BYTES);
#pragma unroll
          for (int hs = 0; hs < 2; ++hs) {
            mbar_wait(&p_full[hs * 2 + b], (pcons >> 1) & 1);
            if (mt == 0 && hs == 0) TRACE(128 + t);
            tc_fence_after();
            const uint32_t p_tm = tmem + hs * 128 + b * 64;
            const uint32_t o_tm = tmem + 256 + hs * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k) {   // 16 keys (8 packed fp16 columns) per k-step
              const uint64_t bd = umma_desc_mn_sw128(vaddr + hs * 8192 + k * 2048, 128 * 128);
              tc_mma_ts(o_tm, p_tm + k * 8, bd, id_pv, (t | k) != 0);
            }
            tc_commit(&pv_done[hs * 2 + b]);
          }
          tc_commit(&kv_empty[stage]);
          ++pcons;
          stage = nst;
          phase = nph;
        }
        tc_commit(o_full);
        tc_commit(q_empty);
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax + epilogue
    // warps 2..9: stream hs = (warp-2)/4 owns keys [64hs, 64hs+64) of every KV tile with its own
    // running max m, sum l and accumulator O_hs (an in-CTA 2-way KV split: the two streams never
    // synchronise per tile, so the 2 warps sharing an SM sub-partition overlap each other's
    // TMEM/MUFU latencies).  Both streams of a row live in the same TMEM lane quarter.
    const int hs = (warp - 2) >> 2;
    const int q = warp & 3;                   // TMEM lane quarter
    const int rl = q * 32 + lane;             // row within the M-tile (= TMEM lane)
    const int et = threadIdx.x - 64;          // 0..255
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t s_base = tmem + hs * 128 + lane_off;
    const uint32_t o_own = tmem + 256 + hs * 128 + lane_off;
    const float sl2 = a.scale_log2;
#define FTRACE(k) \
  do {            \
    if (et == 0 && mt < 2 && t < 16) TRACE((mt ? 448 : 384) + 4 * t + (k)); \
  } while (0)
    uint32_t scons = 0;   // S tiles consumed (all passes)
    for (int mt = 0; mt < n_mt; ++mt) {
      const int rows_mt = min(spm, S - mt * spm) * G;   // valid rows in this M-tile
      const bool valid_row = rl < rows_mt;
      const int slot = mt * spm + rl / G;
      const int j = rl % G;
      const uint64_t anc = (valid_row && slot > 0) ? s_anc[slot] : 0ull;
      float m_used = -INFINITY, l = 0.f;
      for (int t = 0; t < ntiles; ++t, ++scons) {
        const uint32_t b = scons & 1;
        const uint32_t s_tm = s_base + b * 64;
        mbar_wait(&s_full[hs * 2 + b], (scons >> 1) & 1);
        if (mt == 0 && et == 0) TRACE(192 + t);
        tc_fence_after();
        const int tt = tile_of(mt, t);
        const bool tree = tt >= n_prefix_tiles;
        // 64-bit visibility mask of my stream's keys in this tile
        uint32_t mk[2] = {0u, 0u};
        if (valid_row) {
          if (!tree) {
            const int key0 = (p_begin + 2 * tt) * 64;
            int kvalid = min(128, L - key0);
            if (p_begin + 2 * tt + 1 >= p_end) kvalid = min(kvalid, 64);
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              const int n = kvalid - 64 * hs - 32 * w;
              mk[w] = n >= 32 ? 0xFFFFFFFFu : (n <= 0 ? 0u : ((1u << n) - 1u));
            }
          } else {
            // key 0 = root, key k >= 1 = node k-1: visible iff root or ancestor-or-self of my node
            const uint64_t lo = slot > 0 ? ((anc << 1) | 1ull) : 1ull;
            const uint32_t w0 = hs ? (slot > 0 ? (uint32_t)(anc >> 63) : 0u) : (uint32_t)lo;
            const uint32_t w1 = hs ? 0u : (uint32_t)(lo >> 32);
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              const int n = S - 64 * hs - 32 * w;
              mk[w] = (w ? w1 : w0) & (n >= 32 ? 0xFFFFFFFFu : (n <= 0 ? 0u : ((1u << n) - 1u)));
            }
          }
        }
        const bool any0 = __any_sync(0xffffffffu, mk[0] != 0u);
        const bool any1 = __any_sync(0xffffffffu, mk[1] != 0u);
        const bool full = __all_sync(0xffffffffu, (mk[0] & mk[1]) == 0xFFFFFFFFu);
        if (any0 || any1) {
          uint32_t sv[64];
          tmem_ld_32x32b_x32(s_tm, *reinterpret_cast<uint32_t(*)[32]>(sv));
          tmem_ld_32x32b_x32(s_tm + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
          tmem_ld_wait();
          FTRACE(0);
          float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
          if (full) {
#pragma unroll
            for (int e = 0; e < 64; e += 4) {
              m0 = fmaxf(m0, __uint_as_float(sv[e]));
              m1 = fmaxf(m1, __uint_as_float(sv[e + 1]));
              m2 = fmaxf(m2, __uint_as_float(sv[e + 2]));
              m3 = fmaxf(m3, __uint_as_float(sv[e + 3]));
            }
          } else {
#pragma unroll
            for (int e = 0; e < 64; ++e)
              m0 = fmaxf(m0, ((mk[e >> 5] >> (e & 31)) & 1u) ? __uint_as_float(sv[e]) : -INFINITY);
          }
          const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * sl2;
          FTRACE(1);
          float alpha = 1.f;
          bool rescale = false;
          if (mx > m_used + 8.f || (m_used == -INFINITY && mx > -INFINITY)) {
            alpha = m_used == -INFINITY ? 0.f : ex2f(m_used - mx);
            rescale = t > 0 && m_used != -INFINITY;
            l *= alpha;
            m_used = mx;
          }
          const float mb = m_used == -INFINITY ? 0.f : m_used;
          // P = 2^(s*scale - m) as packed fp16 pairs: my 64 keys -> columns [0, 32) of the buffer
          float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t pk[16];
            if (full) {
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const float p0 = ex2f(fmaf(__uint_as_float(sv[32 * c + e]), sl2, -mb));
                const float p1 = ex2f(fmaf(__uint_as_float(sv[32 * c + e + 1]), sl2, -mb));
                ls0 += p0;
                ls1 += p1;
                pk[e >> 1] = pack2(p0, p1);
              }
            } else if (c ? any1 : any0) {
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const float p0 = ((mk[c] >> e) & 1u) ? ex2f(fmaf(__uint_as_float(sv[32 * c + e]), sl2, -mb)) : 0.f;
                const float p1 = ((mk[c] >> (e + 1)) & 1u) ? ex2f(fmaf(__uint_as_float(sv[32 * c + e + 1]), sl2, -mb)) : 0.f;
                ls0 += p0;
                ls1 += p1;
                pk[e >> 1] = pack2(p0, p1);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) pk[e] = 0u;
            }
            tmem_st_32x32b_x16(s_tm + 16 * c, pk);
          }
          l += ls0 + ls1;
          FTRACE(2);
          if (__any_sync(0xffffffffu, rescale)) {
            // O_hs *= alpha: PV_hs(t-1) writes O_hs and may still be in flight -> wait for it
            const uint32_t pb = (scons - 1) & 1;
            mbar_wait(&pv_done[hs * 2 + pb], ((scons - 1) >> 1) & 1);
            tc_fence_after();
            if (rescale) {
#pragma unroll 1
              for (int c = 0; c < HD / 32; ++c) {
                uint32_t ov[32];
                tmem_ld_32x32b_x32(o_own + c * 32, ov);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
                tmem_st_32x32b_x32(o_own + c * 32, ov);
              }
            }
          }
        } else {
          // no visible key of my stream for any row of this warp: P = 0
          uint32_t z[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) z[e] = 0u;
          tmem_st_32x32b_x16(s_tm, z);
          tmem_st_32x32b_x16(s_tm + 16, z);
        }
        tmem_st_wait();
        FTRACE(3);
        if (mt == 0 && et == 0) TRACE(256 + t);
        tc_fence_before();
        mbar_arrive(&p_full[hs * 2 + b]);
      }
      // epilogue: merge the two streams (m_h, l_h, O_h) of every row; warp (q, hs) writes the
      // head-dim columns [hs*HD/2, hs*HD/2 + HD/2)
      s_ml[hs * 256 + rl] = m_used;
      s_ml[hs * 256 + 128 + rl] = l;
      mbar_wait(o_full, mt & 1);
      if (mt == 0 && et == 0) TRACE(320);
      tc_fence_after();
      named_bar_sync(2, 256);
      const float ma = s_ml[rl], mbv = s_ml[256 + rl];
      const float ms = fmaxf(ma, mbv);
      const float c0 = ma == -INFINITY ? 0.f : ex2f(ma - ms);
      const float c1 = mbv == -INFINITY ? 0.f : ex2f(mbv - ms);
      const float lt = s_ml[128 + rl] * c0 + s_ml[384 + rl] * c1;
      const size_t rh = (size_t)(row0 + slot) * a.H + (size_t)g * G + j;
      const bool single = a.n_splits == 1;
      const float inv = single ? (lt > 0.f ? 1.f / lt : 0.f) : 1.f;
      const float f0 = c0 * inv, f1 = c1 * inv;
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        const int col = hs * (HD / 2) + c * 32;
        uint32_t oa[32], ob[32];
        tmem_ld_32x32b_x32(tmem + 256 + lane_off + col, oa);
        tmem_ld_32x32b_x32(tmem + 384 + lane_off + col, ob);
        tmem_ld_wait();
        float ov[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) ov[e] = __uint_as_float(oa[e]) * f0 + __uint_as_float(ob[e]) * f1;
        if (valid_row) {
          if (single) {
            if (ta.O) {
              uint4* dst = reinterpret_cast<uint4*>(ta.O + rh * HD + col);
#pragma unroll
              for (int e = 0; e < 32; e += 8)
                dst[e / 8] = make_uint4(pack2_bf16(ov[e], ov[e + 1]), pack2_bf16(ov[e + 2], ov[e + 3]),
                                        pack2_bf16(ov[e + 4], ov[e + 5]), pack2_bf16(ov[e + 6], ov[e + 7]));
            }
            if (ta.O_f32) {
              float4* dst = reinterpret_cast<float4*>(ta.O_f32 + rh * HD + col);
#pragma unroll
              for (int e = 0; e < 32; e += 4) dst[e / 4] = make_float4(ov[e], ov[e + 1], ov[e + 2], ov[e + 3]);
            }
          } else {
            float4* dst = reinterpret_cast<float4*>(a.opart + ((size_t)sp * a.R * a.H + rh) * HD + col);
#pragma unroll
            for (int e = 0; e < 32; e += 4) dst[e / 4] = make_float4(ov[e], ov[e + 1], ov[e + 2], ov[e + 3]);
          }
        }
      }
      if (valid_row && !single && hs == 0) {
        a.mpart[(size_t)sp * a.R * a.H + rh] = ms;
        a.lpart[(size_t)sp * a.R * a.H + rh] = lt;
      }
      tc_fence_before();
      mbar_arrive(o_empty);
      named_bar_sync(2, 256);   // s_ml reuse by the next pass
    }
  }
  __syncthreads();
  TRACE(321);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

bool tmap_rows(CUtensorMap* m, const void* base, uint64_t rows, int hd) {
  cuuint64_t dims[2] = {(cuuint64_t)hd, rows};
  cuuint64_t strides[1] = {(cuuint64_t)hd * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tmap_q(CUtensorMap* m, const void* base, uint64_t R, int H, int hd, int G, int spm) {
  cuuint64_t dims[3] = {(cuuint64_t)hd, (cuuint64_t)H, R};
  cuuint64_t strides[2] = {(cuuint64_t)hd * 2, (cuuint64_t)H * hd * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)G, (cuuint32_t)spm};
  cuuint32_t estr[3] = {1, 1, 1};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD>
cudaError_t launch_tc(const AttnArgs& a, int B, bf16* O, float* O_f32, cudaStream_t st) {
  CUtensorMap tq, tp, tt;
  const int spm = 128 / a.G;
  const uint64_t pool_rows = (uint64_t)(a.layer + 1) * a.num_pages * 2 * a.KV * 64;
  const uint64_t tree_rows = (uint64_t)(a.layer + 1) * 2 * a.KV * a.R_cap;
  if (!encode_fn() || !tmap_q(&tq, a.Q, (uint64_t)a.R, a.H, HD, a.G, spm) || !tmap_rows(&tp, a.pool, pool_rows, HD) ||
      !tmap_rows(&tt, a.tree_kv, tree_rows, HD))
    return cudaErrorInvalidValue;
  static unsigned long long* trace = nullptr;
  if (getenv("SPECEDGE_ATTN_TRACE") && !trace) cudaMalloc(&trace, 512 * 8);
  TcArgs ta{a, O, O_f32, spm, trace};
  const size_t smem = (size_t)128 * HD * 2 * (1 + 2 * kStages) + 8 * 24 + 66 * 8 + 512 * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(B * a.KV, a.n_splits);
  if (trace) cudaMemsetAsync(trace, 0, 512 * 8, st);
  k_attn_tc<HD><<<grid, kThreads, smem, st>>>(tq, tp, tt, ta);
  if (trace) {
    static int calls = 0;
    unsigned long long h[512];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
    if (++calls % 32 == 5) {   // one layer per step
      const unsigned long long t0 = h[322];
      auto d = [&](int i) { return h[i] ? (long long)(h[i] - t0) : -1LL; };
      fprintf(stderr, "attn trace (cycles from start): end=%lld o_full=%lld\n", d(321), d(320));
      for (int t = 0; t < 12; ++t)
        fprintf(stderr, "  tile %2d: tma_issued=%7lld s_ready(wg0)=%7lld p_done(wg0)=%7lld mma_got_p0=%7lld\n", t, d(t),
                d(192 + t), d(256 + t), d(128 + t));
      for (int m = 0; m < 2; ++m)
        for (int t = 0; t < 10; ++t) {
          const int b = (m ? 448 : 384) + 4 * t;
          fprintf(stderr, "  pass %d tile %2d: ld=%7lld bar=%7lld exp=%7lld st=%7lld\n", m, t, d(b), d(b + 1), d(b + 2),
                  d(b + 3));
        }
    }
  }
  return cudaGetLastError();
}

}  // namespace

unsigned long long* attention_tc_trace_ptr() {
  static unsigned long long* p = nullptr;
  return p;
}

bool attention_tc_supported(int hd, int G) { return (hd == 64 || hd == 128) && G >= 1 && G <= 128; }

cudaError_t attention_tc_launch(const AttnArgs& a, int B, bf16* O, float* O_f32, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  if (a.hd == 128) return launch_tc<128>(a, B, O, O_f32, st);
  if (a.hd == 64) return launch_tc<64>(a, B, O, O_f32, st);
  return cudaErrorInvalidValue;
}

}  // namespace se
