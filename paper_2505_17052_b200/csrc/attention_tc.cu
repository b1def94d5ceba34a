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

namespace se {

namespace {

constexpr int kWarps = 10;
constexpr int kThreads = kWarps * 32;

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
};

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmPool,
              const __grid_constant__ CUtensorMap tmTree, const __grid_constant__ TcArgs ta) {
  constexpr int KB = HD / 64;                  // 64-element hd blocks
  constexpr uint32_t QT_BYTES = 128 * HD * 2;  // one M-tile of Q
  constexpr uint32_t KT_BYTES = 128 * HD * 2;  // one 128-key tile of K (or V)
  const AttnArgs& a = ta.a;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                              // [2][KB][128 rows][128 B]
  uint8_t* sK = sQ + 2 * QT_BYTES;                 // [2 stages][KB][128 keys][128 B]
  uint8_t* sV = sK + 2 * KT_BYTES;                 // [2 stages][KB][128 keys][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * KT_BYTES);
  uint64_t* q_full = bars;          // [1]
  uint64_t* q_empty = bars + 1;     // [1]
  uint64_t* kv_full = bars + 2;     // [2]
  uint64_t* kv_empty = bars + 4;    // [2]
  uint64_t* s_full = bars + 6;      // [2]
  uint64_t* p_full = bars + 8;      // [2]
  uint64_t* o_full = bars + 10;     // [2]
  uint64_t* o_empty = bars + 12;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  uint64_t* s_anc = reinterpret_cast<uint64_t*>(bars + 16);   // [65]

  const int r = blockIdx.x / a.KV, g = blockIdx.x % a.KV, sp = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
  const int S = min(a.req_S[r], a.max_rows / G);
  const int L = a.req_L[r];
  const int row0 = a.req_row0[r];
  const int h = a.req_h[r];
  const int spm = ta.slots_per_mt;
  const int n_mt = (S + spm - 1) / spm;
  const int npages = (L + 63) / 64;
  const int p_begin = sp * a.pages_per_split;
  const int p_end = min(npages, p_begin + a.pages_per_split);
  const int n_prefix_tiles = max(0, (p_end - p_begin + 1) / 2);
  const bool has_tree = sp == a.n_splits - 1;
  const int ntiles = n_prefix_tiles + (has_tree ? 1 : 0);
  const int n_pairs = (n_mt + 1) / 2;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmPool);
    tma_prefetch(&tmTree);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 128);
    }
    fence_barrier_init();
  }
  for (int s = threadIdx.x; s < S && s <= kMaxNodes; s += blockDim.x) s_anc[s] = a.row_anc[row0 + s];
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------------- TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int pr = 0; pr < n_pairs; ++pr) {
        mbar_wait(q_empty, (pr & 1) ^ 1);
        const int nm = min(2, n_mt - 2 * pr);
        const uint32_t qbox = (uint32_t)(64 * G * spm * 2);
        mbar_expect_tx(q_full, qbox * KB * nm);
        for (int mi = 0; mi < nm; ++mi)
          for (int kb = 0; kb < KB; ++kb)
            tma_load_3d(sQ + mi * QT_BYTES + kb * 128 * 128, &tmQ, q_full, kb * 64, g * G,
                        row0 + (2 * pr + mi) * spm);
        for (int t = 0; t < ntiles; ++t) {
          mbar_wait(&kv_empty[stage], phase ^ 1);
          mbar_expect_tx(&kv_full[stage], 2 * KT_BYTES);
          uint8_t* dk = sK + stage * KT_BYTES;
          uint8_t* dv = sV + stage * KT_BYTES;
          if (t < n_prefix_tiles) {
            for (int half = 0; half < 2; ++half) {
              int p = p_begin + 2 * t + half;
              if (p >= p_end) p = p_begin + 2 * t;   // odd tail: reload a valid page, masked later
              const int page = a.block_table[(size_t)h * a.max_pages_per_seq + p];
              const int rk = (((a.layer * a.num_pages + page) * 2 + 0) * a.KV + g) * 64;
              const int rv = rk + a.KV * 64;
              for (int kb = 0; kb < KB; ++kb) {
                tma_load_2d(dk + kb * 128 * 128 + half * 64 * 128, &tmPool, &kv_full[stage], kb * 64, rk);
                tma_load_2d(dv + kb * 128 * 128 + half * 64 * 128, &tmPool, &kv_full[stage], kb * 64, rv);
              }
            }
          } else {
            const int rk = ((a.layer * 2 + 0) * a.KV + g) * a.R_cap + row0;
            const int rv = ((a.layer * 2 + 1) * a.KV + g) * a.R_cap + row0;
            for (int half = 0; half < 2; ++half)
              for (int kb = 0; kb < KB; ++kb) {
                tma_load_2d(dk + kb * 128 * 128 + half * 64 * 128, &tmTree, &kv_full[stage], kb * 64, rk + 64 * half);
                tma_load_2d(dv + kb * 128 * 128 + half * 64 * 128, &tmTree, &kv_full[stage], kb * 64, rv + 64 * half);
              }
          }
          if (++stage == 2) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------------- MMA issuer
    if (elect_one()) {
      const uint32_t id_qk = idesc_f16(128, 128, false);
      const uint32_t id_pv = idesc_f16(128, HD, true);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t sp_phase[2] = {0, 0};
      for (int pr = 0; pr < n_pairs; ++pr) {
        const int nm = min(2, n_mt - 2 * pr);
        mbar_wait(q_full, pr & 1);
        // the epilogue of the previous pair must have drained O before it is re-initialised
        for (int mi = 0; mi < nm; ++mi) mbar_wait(&o_empty[mi], (pr & 1) ^ 1);
        tc_fence_after();
        // S_m(t+1) is issued right behind PV_m(t) so that the softmax of tile t+1 for one M-tile
        // overlaps the MMAs and softmax of the other (tcgen05.mma executes in issue order, so
        // S_m(t+1) cannot overwrite P_m(t) before PV_m(t) has read it).
        auto issue_qk = [&](int mi, uint32_t kaddr) {
          const uint32_t qaddr = smem_u32(sQ + mi * QT_BYTES);
          const uint32_t s_tm = tmem + mi * 256;
#pragma unroll
          for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16(s_tm, umma_desc_sw128(qaddr + kb * 16384 + k * 32), umma_desc_sw128(kaddr + kb * 16384 + k * 32),
                         id_qk, (kb | k) != 0);
          tc_commit(&s_full[mi]);
        };
        if (ntiles > 0) {
          mbar_wait(&kv_full[stage], phase);
          tc_fence_after();
          for (int mi = 0; mi < nm; ++mi) issue_qk(mi, smem_u32(sK + stage * KT_BYTES));
        }
        for (int t = 0; t < ntiles; ++t) {
          const int nstage = stage ^ 1;
          const uint32_t nphase = phase ^ (stage == 1 ? 1u : 0u);
          const uint32_t vaddr = smem_u32(sV + stage * KT_BYTES);
          for (int mi = 0; mi < nm; ++mi) {
            mbar_wait(&p_full[mi], sp_phase[mi]);
            sp_phase[mi] ^= 1;
            tc_fence_after();
            const uint32_t p_tm = tmem + mi * 256;
            const uint32_t o_tm = tmem + mi * 256 + 128;
#pragma unroll
            for (int k = 0; k < 8; ++k) {   // 16 keys (8 packed fp16 columns) per k-step
              const uint64_t bd = umma_desc_mn_sw128(vaddr + k * 2048, 128 * 128);
              tc_mma_ts(o_tm, p_tm + k * 8, bd, id_pv, (t | k) != 0);
            }
            if (mi == nm - 1) tc_commit(&kv_empty[stage]);
            if (t + 1 < ntiles) {
              if (mi == 0) {
                mbar_wait(&kv_full[nstage], nphase);
                tc_fence_after();
              }
              issue_qk(mi, smem_u32(sK + nstage * KT_BYTES));
            }
          }
          stage = nstage;
          phase = nphase;
        }
        for (int mi = 0; mi < nm; ++mi) tc_commit(&o_full[mi]);
        tc_commit(q_empty);
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax + epilogue
    const int wg = (warp - 2) >> 2;           // M-tile slot of this warpgroup
    const int q = warp & 3;                   // TMEM lane quarter
    const int rl = q * 32 + lane;             // row within the M-tile (= TMEM lane)
    const float sl2 = a.scale_log2;
    uint32_t s_phase = 0;
    for (int pr = 0; pr < n_pairs; ++pr) {
      const int mt = 2 * pr + wg;
      const bool active_mt = mt < n_mt;
      if (!active_mt) continue;
      const int rows_mt = min(spm, S - mt * spm) * G;   // valid rows in this M-tile
      const bool valid_row = rl < rows_mt;
      const int slot = mt * spm + rl / G;
      const int j = rl % G;
      const uint64_t anc = (valid_row && slot > 0) ? s_anc[slot] : 0ull;
      const uint32_t s_tm = tmem + wg * 256 + ((uint32_t)(q * 32) << 16);
      const uint32_t o_tm = s_tm + 128;
      float m_used = -INFINITY, l = 0.f;
      for (int t = 0; t < ntiles; ++t) {
        mbar_wait(&s_full[wg], s_phase);
        s_phase ^= 1;
        tc_fence_after();
        const bool tree = t >= n_prefix_tiles;
        // 128-bit visibility mask of this tile's keys for this row
        uint32_t mk[4] = {0u, 0u, 0u, 0u};
        if (valid_row) {
          if (!tree) {
            const int key0 = (p_begin + 2 * t) * 64;
            int kvalid = min(128, L - key0);
            if (p_begin + 2 * t + 1 >= p_end) kvalid = min(kvalid, 64);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const int n = kvalid - 32 * w;
              mk[w] = n >= 32 ? 0xFFFFFFFFu : (n <= 0 ? 0u : ((1u << n) - 1u));
            }
          } else {
            // key 0 = root, key k >= 1 = node k-1: visible iff root or ancestor-or-self of my node
            const uint64_t lo = slot > 0 ? ((anc << 1) | 1ull) : 1ull;
            mk[0] = (uint32_t)lo;
            mk[1] = (uint32_t)(lo >> 32);
            mk[2] = slot > 0 ? (uint32_t)(anc >> 63) : 0u;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const int n = S - 32 * w;
              mk[w] &= n >= 32 ? 0xFFFFFFFFu : (n <= 0 ? 0u : ((1u << n) - 1u));
            }
          }
        }
        const bool any_valid = __any_sync(0xffffffffu, (mk[0] | mk[1] | mk[2] | mk[3]) != 0u);
        if (any_valid) {
          // the whole row of 128 scores in registers
          uint32_t sv[128];
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(s_tm + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32 * c));
          tmem_ld_wait();
          const bool full = __all_sync(0xffffffffu, (mk[0] & mk[1] & mk[2] & mk[3]) == 0xFFFFFFFFu);
          float mx = -INFINITY;
          if (full) {
#pragma unroll
            for (int e = 0; e < 128; ++e) mx = fmaxf(mx, __uint_as_float(sv[e]));
          } else {
#pragma unroll
            for (int e = 0; e < 128; ++e)
              mx = fmaxf(mx, ((mk[e >> 5] >> (e & 31)) & 1u) ? __uint_as_float(sv[e]) : -INFINITY);
          }
          mx *= sl2;
          float alpha = 1.f;
          bool rescale = false;
          if (mx > m_used + 8.f || (m_used == -INFINITY && mx > -INFINITY)) {
            alpha = m_used == -INFINITY ? 0.f : ex2f(m_used - mx);
            rescale = t > 0 && m_used != -INFINITY;
            l *= alpha;
            m_used = mx;
          }
          const float mb = m_used == -INFINITY ? 0.f : m_used;
          // P = 2^(s*scale - m) as packed fp16 pairs into the first 64 columns of this S region,
          // 32 keys (16 columns) at a time (column 16c <= 32c: never overwrites unread scores)
          float ls = 0.f;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t pk[16];
            if (full) {
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const float p0 = ex2f(fmaf(__uint_as_float(sv[32 * c + e]), sl2, -mb));
                const float p1 = ex2f(fmaf(__uint_as_float(sv[32 * c + e + 1]), sl2, -mb));
                ls += p0 + p1;
                pk[e >> 1] = pack2(p0, p1);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const float p0 = ((mk[c] >> e) & 1u) ? ex2f(fmaf(__uint_as_float(sv[32 * c + e]), sl2, -mb)) : 0.f;
                const float p1 = ((mk[c] >> (e + 1)) & 1u) ? ex2f(fmaf(__uint_as_float(sv[32 * c + e + 1]), sl2, -mb)) : 0.f;
                ls += p0 + p1;
                pk[e >> 1] = pack2(p0, p1);
              }
            }
            tmem_st_32x32b_x16(s_tm + 16 * c, pk);
          }
          l += ls;
          if (rescale) {
            // O *= alpha before PV of this tile (PV of tile t-1 is complete: s_full of this tile
            // was committed after it)
#pragma unroll 1
            for (int c = 0; c < HD / 32; ++c) {
              uint32_t ov[32];
              tmem_ld_32x32b_x32(o_tm + c * 32, ov);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
              tmem_st_32x32b_x32(o_tm + c * 32, ov);
            }
          }
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[wg]);
      }
      // epilogue: O of this M-tile
      mbar_wait(&o_full[wg], pr & 1);
      tc_fence_after();
      const size_t rh = (size_t)(row0 + slot) * a.H + (size_t)g * G + j;
      const bool single = a.n_splits == 1;
      const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t ov[32];
        tmem_ld_32x32b_x32(o_tm + c * 32, ov);
        tmem_ld_wait();
        if (valid_row) {
          if (single) {
            if (ta.O) {
              uint4* dst = reinterpret_cast<uint4*>(ta.O + rh * HD + c * 32);
#pragma unroll
              for (int e = 0; e < 32; e += 8)
                dst[e / 8] = make_uint4(pack2_bf16(__uint_as_float(ov[e]) * inv, __uint_as_float(ov[e + 1]) * inv),
                                        pack2_bf16(__uint_as_float(ov[e + 2]) * inv, __uint_as_float(ov[e + 3]) * inv),
                                        pack2_bf16(__uint_as_float(ov[e + 4]) * inv, __uint_as_float(ov[e + 5]) * inv),
                                        pack2_bf16(__uint_as_float(ov[e + 6]) * inv, __uint_as_float(ov[e + 7]) * inv));
            }
            if (ta.O_f32) {
              float4* dst = reinterpret_cast<float4*>(ta.O_f32 + rh * HD + c * 32);
#pragma unroll
              for (int e = 0; e < 32; e += 4)
                dst[e / 4] = make_float4(__uint_as_float(ov[e]) * inv, __uint_as_float(ov[e + 1]) * inv,
                                         __uint_as_float(ov[e + 2]) * inv, __uint_as_float(ov[e + 3]) * inv);
            }
          } else {
            float4* dst = reinterpret_cast<float4*>(a.opart + ((size_t)sp * a.R * a.H + rh) * HD + c * 32);
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              dst[e / 4] = make_float4(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1]), __uint_as_float(ov[e + 2]),
                                       __uint_as_float(ov[e + 3]));
          }
        }
      }
      if (valid_row && !single) {
        a.mpart[(size_t)sp * a.R * a.H + rh] = m_used;
        a.lpart[(size_t)sp * a.R * a.H + rh] = l;
      }
      tc_fence_before();
      mbar_arrive(&o_empty[wg]);
    }
  }
  __syncthreads();
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
  TcArgs ta{a, O, O_f32, spm};
  const size_t smem = 1024 + 2 * (size_t)128 * HD * 2 * 3 + 16 * 8 + 66 * 8 + 64;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(B * a.KV, a.n_splits);
  k_attn_tc<HD><<<grid, kThreads, smem, st>>>(tq, tp, tt, ta);
  return cudaGetLastError();
}

}  // namespace

bool attention_tc_supported(int hd, int G) { return (hd == 64 || hd == 128) && G >= 1 && G <= 128; }

cudaError_t attention_tc_launch(const AttnArgs& a, int B, bf16* O, float* O_f32, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  if (a.hd == 128) return launch_tc<128>(a, B, O, O_f32, st);
  if (a.hd == 64) return launch_tc<64>(a, B, O, O_f32, st);
  return cudaErrorInvalidValue;
}

}  // namespace se
