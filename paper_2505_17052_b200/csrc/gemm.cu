// tcgen05 / TMEM / TMA GEMM with fused epilogues for the verify step's dense contractions
// (QKV, O-proj, gate/up + SwiGLU, down, LM head + vocab argmax /
// Gumbel-max).  O / down (and QKV when it must be K-split) store fp32 per-K-split partials, summed
// in a fixed order (deterministic) by the following elementwise kernels (kernels_small.cu: the
// residual add + RMSNorm, or RoPE + K/V scatter); an unsplit QKV GEMM applies RoPE and the K/V
// scatter in its own epilogue (EPI_QKV).  P:173 ("a single forward pass" over
// all draft tokens) makes these weight-streaming GEMMs with N = R rows of the whole batch.
//
// Orientation ("swap-AB"): D^T[feature][row] = W[feature][:] . X[row][:].  Weights take the
// MMA's M = 128 side (always a multiple of 128 after zero-fill), the R activation rows of the
// batch take N = BN <= 256 (multiple of 16), so ragged small R wastes < 16 rows per tile.
// Both operands are K-major bf16, TMA-loaded with 128B swizzle into a `stages`-deep ring;
// one elected thread issues tcgen05.mma (fp32 accumulators in TMEM, double-buffered so the
// epilogue of tile i overlaps the MMAs of tile i+1); four epilogue warps read TMEM with
// tcgen05.ld and apply the fused epilogue.  Persistent grid: one CTA per SM, static stride.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <cstdlib>

namespace se {

namespace {

// warp 0 TMA, warp 1 MMA + TMEM alloc, warps 2..9 epilogue in kEpiGroups groups of four warps
// (one per TMEM lane quarter each): group g takes the accumulator's 32-column chunks c = g mod 2,
// with its own exchange / reduction buffers and named barrier 1 + g, so a tile's epilogue (the
// unoverlapped tail of every GEMM launch) runs on twice the warps
constexpr int kEpiGroups = 2;
constexpr int kEpiThreads = 128;        // per group
constexpr int kThreads = 64 + kEpiGroups * kEpiThreads;
constexpr uint32_t kXchBytes = 128 * 33 * 4;
constexpr uint32_t kRedBytes = 4 * 32 * 24;
constexpr uint32_t kABytes = 128 * 128;  // 128 rows x 64 bf16
constexpr int kXchStride = 33;


struct SmemLayout {
  uint32_t a_off, b_off, xch_off, red_off, bar_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(int stages, int BN) {
  SmemLayout L;
  L.a_off = 0;
  L.b_off = L.a_off + stages * kABytes;
  L.xch_off = L.b_off + stages * (uint32_t)BN * 128u;   // [kEpiGroups][kXchBytes]
  L.red_off = L.xch_off + kEpiGroups * kXchBytes;          // [kEpiGroups][kRedBytes]: red_v, red_i [128];
                                                           // top2: red_s2, red_i2 at +256, red_s3 at +512;
                                                           // noise row inputs at +640 (128 words)
  L.bar_off = L.red_off + kEpiGroups * kRedBytes;
  L.total = L.bar_off + (2 * stages + 4) * 8 + 16;
  return L;
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + expf(-g)); }
__device__ __forceinline__ uint32_t pack2_f16(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack2_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Epilogue of one 32-column chunk of a 128-feature accumulator tile.  v[j] = D[feature][row]
// for feature = m128*128 + tl (tl = TMEM lane) and row = row_base + j, j < ncol.
template <int MODE>
__device__ __forceinline__ void epi_chunk(const GemmArgs& a, const uint32_t (&v)[32], int m128, int tl, int et,
                                          int row_base, int ncol, int sk, float* xch, float* red_v, int* red_i,
                                          int bar) {
    const int feat = m128 * 128 + tl;
    if constexpr (MODE == EPI_F32) {
      if (a.push) {
        // NEXT-F4 push: stage the chunk row-major (32 rows x 128 features = 32 x 512 B), then
        // one lane per warp sends 8 rows to their owners' receive slots with bulk async copies
        // (remote rows cross NVLink) — the epilogue warps never wait on a remote store.  Every
        // epilogue thread reaches both barriers (lanes past M stage zeros); a copy carries only
        // the tile's features below M.
        for (int j = 0; j < 32; ++j) xch[j * 128 + tl] = feat < a.M ? __uint_as_float(v[j]) : 0.f;
        fence_proxy_async_smem();
        named_bar_sync(bar, kEpiThreads);
        const uint32_t nbytes = (uint32_t)min(128, a.M - m128 * 128) * 4u;
        if ((et & 31) == 0) {   // one issuing lane per epilogue warp, 8 rows each
          for (int j = (et >> 5) * 8; j < min(ncol, (et >> 5) * 8 + 8); ++j) {
            const int row = row_base + j;
            if (row >= a.R) break;
            const int o = row / a.rows_per_rank;
            bulk_s2g(a.peer_out[o] + (size_t)a.tp_src * a.slot_stride + (size_t)(row - o * a.rows_per_rank) * a.ldo +
                         m128 * 128,
                     xch + j * 128, nbytes);
          }
          bulk_commit();
          bulk_wait_read0();   // the staging buffer may be overwritten
        }
        named_bar_sync(bar, kEpiThreads);
      } else if (feat < a.M) {
        if (a.pair) {   // physical rows 2r, 2r+1 hold hi/lo parts of logical row r
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const int row = row_base + j;
            if (j < ncol && row < a.R)
              a.out_f32[(size_t)(row >> 1) * a.ldo + feat] = __uint_as_float(v[j]) + __uint_as_float(v[j + 1]);
          }
        } else if (a.resid && a.splits == 1) {   // fused residual add, unsplit: X + Y0
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int row = row_base + j;
            if (j < ncol && row < a.R) {
              float* x = a.resid + (size_t)row * a.ldo + feat;
              *x = *x + __uint_as_float(v[j]);
            }
          }
        } else {
          float* out = a.out_f32 + (size_t)sk * a.split_stride;   // K-split sk's partial
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int row = row_base + j;
            if (j < ncol && row < a.R) out[(size_t)row * a.ldo + feat] = __uint_as_float(v[j]);
          }
        }
      }
    } else if constexpr (MODE == EPI_SWIGLU) {
      // tile rows: lanes 0..63 = gate features m*64 + i, lanes 64..127 = up features
#pragma unroll
      for (int j = 0; j < 32; ++j) xch[tl * kXchStride + j] = __uint_as_float(v[j]);
      named_bar_sync(bar, kEpiThreads);
      // transposed: item (row j, group i) = output features m*64 + [8i, 8i+8), one 16-B store;
      // the 8 lanes of a row write its 128 contiguous bytes (4 rows per warp instruction)
      const int i = et & 7;
      const int fo = m128 * 64 + 8 * i;
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int j = (et >> 3) + 16 * it;
        const int row = row_base + j;
        if (j < ncol && row < a.R && fo < a.M / 2) {
          float y[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float g = xch[(8 * i + e) * kXchStride + j], u = xch[(8 * i + 64 + e) * kXchStride + j];
            y[e] = silu_f(g) * u;
          }
          *reinterpret_cast<uint4*>(a.out_bf16 + (size_t)row * a.ld_out + fo) =
              make_uint4(pack2_bf16(y[0], y[1]), pack2_bf16(y[2], y[3]), pack2_bf16(y[4], y[5]), pack2_bf16(y[6], y[7]));
        }
      }
      named_bar_sync(bar, kEpiThreads);
    } else if constexpr (MODE == EPI_QKV) {
      // 128-feature tile m128 = one head (head_dim 128): q heads [0, H), k heads [H, H+KV), v
      // heads after.  q / k: rotate-half RoPE at row_pos (pairs (i, i+64) sit in lanes i and
      // i+64, exchanged through shared memory as in the SwiGLU epilogue); v: plain fp16 copy.
      // Same arithmetic and rounding as k_qkv_rope (fp32 in, one fp16 rounding out).
      // The chunk is transposed through shared memory so that every store is 16 B of one row:
      // item (row j, group i) = features [8i, 8i+8) and their rotate-half partners [8i+64, 8i+72);
      // the 8 lanes of a row write its 2 x 128 contiguous bytes (4 rows per warp instruction).
      const int head = m128;
      const int H = a.n_heads, KV = a.n_kv;
      f16* const Qo = reinterpret_cast<f16*>(a.out_bf16);
      f16* const kv = reinterpret_cast<f16*>(a.tree_kv);
      const bool is_v = head >= H + KV;
      f16* const base = head < H ? Qo + (size_t)head * 128
                        : kv + (((size_t)a.layer * 2 + (is_v ? 1 : 0)) * KV + (head - H - (is_v ? KV : 0))) *
                                   a.R_cap * 128;
      const size_t rstride = head < H ? (size_t)H * 128 : 128;
#pragma unroll
      for (int j = 0; j < 32; ++j) xch[tl * kXchStride + j] = __uint_as_float(v[j]);
      named_bar_sync(bar, kEpiThreads);
      const int i = et & 7;
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int j = (et >> 3) + 16 * it;
        const int row = row_base + j;
        if (j < ncol && row < a.R) {
          float x1[8], x2[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            x1[e] = xch[(8 * i + e) * kXchStride + j];
            x2[e] = xch[(8 * i + 64 + e) * kXchStride + j];
          }
          uint4 o1, o2;
          if (is_v) {
            o1 = make_uint4(pack2_f16(x1[0], x1[1]), pack2_f16(x1[2], x1[3]), pack2_f16(x1[4], x1[5]),
                            pack2_f16(x1[6], x1[7]));
            o2 = make_uint4(pack2_f16(x2[0], x2[1]), pack2_f16(x2[2], x2[3]), pack2_f16(x2[4], x2[5]),
                            pack2_f16(x2[6], x2[7]));
          } else {
            const int pos = __ldg(a.row_pos + row);
            const float4* cp = reinterpret_cast<const float4*>(a.rope_cos + (size_t)pos * 64 + 8 * i);
            const float4* sp = reinterpret_cast<const float4*>(a.rope_sin + (size_t)pos * 64 + 8 * i);
            const float4 c0 = __ldg(cp), c1 = __ldg(cp + 1), s0 = __ldg(sp), s1 = __ldg(sp + 1);
            const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            float r1[8], r2[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              r1[e] = x1[e] * cs[e] - x2[e] * sn[e];
              r2[e] = x2[e] * cs[e] + x1[e] * sn[e];
            }
            o1 = make_uint4(pack2_f16(r1[0], r1[1]), pack2_f16(r1[2], r1[3]), pack2_f16(r1[4], r1[5]),
                            pack2_f16(r1[6], r1[7]));
            o2 = make_uint4(pack2_f16(r2[0], r2[1]), pack2_f16(r2[2], r2[3]), pack2_f16(r2[4], r2[5]),
                            pack2_f16(r2[6], r2[7]));
          }
          f16* dst = base + (size_t)row * rstride + 8 * i;
          *reinterpret_cast<uint4*>(dst) = o1;
          *reinterpret_cast<uint4*>(dst + 64) = o2;
        }
      }
      named_bar_sync(bar, kEpiThreads);
    } else if constexpr (MODE == EPI_ARGMAX || MODE == EPI_PQ1 || MODE == EPI_PQ2) {
      // the CTA pair's second 128-feature half past the last vocab tile (an odd tile count, e.g.
      // V = 151936 = 1187 x 128): nothing to reduce, and its partial slot [lr][ntm128] would be
      // the next row's tile 0 (uniform per CTA: every epilogue thread returns, no barrier is split)
      if (m128 >= a.ntm128) return;
      // a.pair: physical rows (2r, 2r+1) = hi/lo parts of logical row r -> 16 logical columns
      const int np = a.pair ? 16 : 32;
      const bool fv = feat < a.vocab;
      const int vg = a.vocab_off + feat;   // global vocab id
      // logical row jj's logit of this thread's feature, or NaN when out of range
      auto logit = [&](int jj, int& lrow) -> float {
        const int j = a.pair ? 2 * jj : jj;
        const int row = row_base + j;
        lrow = a.pair ? row >> 1 : row;
        if (!fv || j >= ncol || row >= a.R) return __int_as_float(0x7fc00000);
        return a.pair ? __uint_as_float(v[2 * jj]) + __uint_as_float(v[2 * jj + 1]) : __uint_as_float(v[jj]);
      };
      // ---- Gumbel noise g(seed, round, session, slot, vg) (SURVEY amb. A9), generated here: no
      // [R][vocab] noise tensor ever reaches HBM.  One Philox4x32-10 block covers 4 consecutive
      // vocab ids = the 4 lanes of a quad (vocab_off % 4 == 0), so lane q of a quad computes the
      // block of logical row j4 + q and stores its 4 words into the quad's 4 cells of that row of
      // the exchange buffer (conflict-free: bank = 4k + q); every lane then reads its own cell.
      // The raw words are turned into noise in the score loop below, which overwrites the cells.
      const bool noisy = MODE == EPI_PQ2 || a.sample;
      const bool quad_ok = (a.vocab_off & 3) == 0;
      // the chunk's per-row Philox inputs (slot, session lo / hi, key word 0), gathered once by the
      // first np threads into the free tail of the reduction area: the dependent row -> request ->
      // session loads would otherwise sit on every lane's critical path
      uint32_t* rinfo = reinterpret_cast<uint32_t*>(red_v + 640);   // [32][4]
      if (noisy) {
        if (et < np) {
          const int j = a.pair ? 2 * et : et;
          const int row = min(row_base + j, a.R - 1);
          const int lr = a.pair ? row >> 1 : row;
          const int req = a.row_req[lr];
          const uint64_t ses = a.req_session[req];
          rinfo[4 * et] = (uint32_t)a.row_slot[lr];
          rinfo[4 * et + 1] = (uint32_t)ses;
          rinfo[4 * et + 2] = (uint32_t)(ses >> 32);
          rinfo[4 * et + 3] = a.seed_lo ^ a.req_round[req];
        }
        named_bar_sync(bar, kEpiThreads);
      }
      if (noisy && quad_ok) {
        const int qd = tl & 3;
        // unrolled: the up to 8 Philox blocks of a lane are independent chains (one epilogue warp
        // per SM sub-partition has no other latency hiding)
#pragma unroll
        for (int j4 = 0; j4 < 32; j4 += 4) {
          if (j4 >= np) break;
          const int jj = j4 + qd;
          const uint4 ri = *reinterpret_cast<const uint4*>(rinfo + 4 * jj);
          const U4 w = philox4x32_10(U4{(uint32_t)vg >> 2, ri.x, ri.y, ri.z}, ri.w, a.seed_hi);
          uint32_t* cell = reinterpret_cast<uint32_t*>(xch) + (tl & ~3) * kXchStride + jj;
          cell[0] = w.x;
          cell[kXchStride] = w.y;
          cell[2 * kXchStride] = w.z;
          cell[3 * kXchStride] = w.w;
        }
        __syncwarp();
      }
      auto gumbel_at = [&](int jj) -> float {
        uint32_t wd;
        if (quad_ok) {
          wd = reinterpret_cast<const uint32_t*>(xch)[tl * kXchStride + jj];
        } else {   // a vocab shard not aligned to 4 ids: this lane's own block
          const uint4 ri = *reinterpret_cast<const uint4*>(rinfo + 4 * jj);
          const U4 w = philox4x32_10(U4{(uint32_t)vg >> 2, ri.x, ri.y, ri.z}, ri.w, a.seed_hi);
          wd = u4_word(w, vg & 3);
        }
        return gumbel_of_word(wd);
      };
      // ---- the chunk's noise first, as 32 independent unrolled chains (the score loop below has
      // data-dependent branches that would serialise the two logf evaluations per value)
      float gn[32];
      if (noisy) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) gn[jj] = gumbel_at(jj);   // rows >= np: unused
      }
      // ---- scores for the tile argmax
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        if (jj >= np) break;
        int lr;
        const float l = logit(jj, lr);
        float sc = -INFINITY;
        if (l == l) {
          if constexpr (MODE == EPI_PQ2) {
            // residual r = p - q (p = exp(l/T - lse)); Gumbel-max over log r, r > 0
            const int qn = a.row_qnode[lr];
            if (qn >= 0) {
              const float pv = __expf(fmaf(l, a.inv_t, -a.lse[lr]));
              if (vg == a.node_token[qn]) a.pchild[lr] = pv;
              const float r = pv - a.draft_q[(size_t)qn * a.vocab_q + vg];
              if (r > 0.f) sc = __logf(r) + gn[jj];
            }
          } else {
            sc = a.sample ? l * a.inv_t + gn[jj] : l;
          }
        }
        xch[tl * kXchStride + jj] = sc;
      }
      named_bar_sync(bar, kEpiThreads);
      const int ngrp = 128 / np, per = 128 / ngrp;
      // tile argmax per row (ties -> lowest id: features scanned in increasing order); a.top2
      // also keeps the tile's second (score, id) and third score (k_lm_refine's candidate window,
      // hi-only pass)
      float* red_s2 = red_v + 256;
      int* red_i2 = red_i + 256;
      float* red_s3 = red_v + 512;
      {
        const int jj = et % np, g = et / np;
        float b1 = -INFINITY, b2 = -INFINITY, b3 = -INFINITY;
        int i1 = 0x7fffffff, i2 = 0x7fffffff;
        for (int l = 0; l < per; ++l) {
          const float sc = xch[(g * per + l) * kXchStride + jj];
          const int id = a.vocab_off + m128 * 128 + g * per + l;
          if (sc > b1) { b3 = b2; b2 = b1; i2 = i1; b1 = sc; i1 = id; }
          else if (sc > b2) { b3 = b2; b2 = sc; i2 = id; }
          else if (sc > b3) b3 = sc;
        }
        red_v[g * np + jj] = b1;
        red_i[g * np + jj] = i1;
        if (a.top2) {
          red_s2[g * np + jj] = b2;
          red_i2[g * np + jj] = i2;
          red_s3[g * np + jj] = b3;
        }
      }
      named_bar_sync(bar, kEpiThreads);
      if (et < np) {
        const int jj = et;
        float b1 = red_v[jj], b2 = -INFINITY, b3 = -INFINITY;
        int i1 = red_i[jj], i2 = 0x7fffffff;
        if (a.top2) { b2 = red_s2[jj]; i2 = red_i2[jj]; b3 = red_s3[jj]; }
        for (int g = 1; g < ngrp; ++g) {
          // merge group g's sorted (b1 >= b2 >= b3) list; groups hold increasing ids, so a tie keeps
          // the earlier (lower) id first
          const float c1 = red_v[g * np + jj];
          const int k1 = red_i[g * np + jj];
          if (!a.top2) {
            if (c1 > b1) { b1 = c1; i1 = k1; }
            continue;
          }
          const float c2 = red_s2[g * np + jj], c3 = red_s3[g * np + jj];
          const int k2 = red_i2[g * np + jj];
          // insert group g's three (its ids are higher: strict > keeps ours first on ties; its own
          // list is in order, so c1 precedes c2 on ties as well)
          auto ins = [&](float val, int id) {
            if (val > b1) { b3 = b2; b2 = b1; i2 = i1; b1 = val; i1 = id; }
            else if (val > b2) { b3 = b2; b2 = val; i2 = id; }
            else if (val > b3) b3 = val;
          };
          ins(c1, k1);
          ins(c2, k2);
          ins(c3, 0x7fffffff);
        }
        const int j = a.pair ? 2 * jj : jj;
        const int row = row_base + j;
        if (j < ncol && row < a.R) {
          const int lr = a.pair ? row >> 1 : row;
          const size_t o = (size_t)lr * a.ntm128 + m128;
          a.part_val[o] = b1;
          a.part_idx[o] = i1;
          if (a.top2) {
            a.part_val2[o] = b2;
            a.part_idx2[o] = i2;
            a.part_val3[o] = b3;
          }
        }
      }
      named_bar_sync(bar, kEpiThreads);
      if constexpr (MODE == EPI_PQ1) {
        // ---- tile (max, sum exp) of l/T for the row's log-sum-exp
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          if (jj >= np) break;
          int lr;
          const float l = logit(jj, lr);
          xch[tl * kXchStride + jj] = l == l ? l * a.inv_t : -INFINITY;
        }
        named_bar_sync(bar, kEpiThreads);
        float* red_s = reinterpret_cast<float*>(red_i);
        {
          const int jj = et % np, g = et / np;
          float m = -INFINITY;
          for (int l = 0; l < per; ++l) m = fmaxf(m, xch[(g * per + l) * kXchStride + jj]);
          float sm = 0.f;
          if (m > -INFINITY)
            for (int l = 0; l < per; ++l) sm += __expf(xch[(g * per + l) * kXchStride + jj] - m);
          red_v[g * np + jj] = m;
          red_s[g * np + jj] = sm;
        }
        named_bar_sync(bar, kEpiThreads);
        if (et < np) {
          const int jj = et;
          float m = -INFINITY;
          for (int g = 0; g < ngrp; ++g) m = fmaxf(m, red_v[g * np + jj]);
          float sm = 0.f;
          if (m > -INFINITY)
            for (int g = 0; g < ngrp; ++g) sm += red_s[g * np + jj] * __expf(red_v[g * np + jj] - m);
          const int j = a.pair ? 2 * jj : jj;
          const int row = row_base + j;
          if (j < ncol && row < a.R) {
            const int lr = a.pair ? row >> 1 : row;
            a.part_m[(size_t)lr * a.ntm128 + m128] = m;
            a.part_s[(size_t)lr * a.ntm128 + m128] = sm;
          }
        }
        named_bar_sync(bar, kEpiThreads);
      }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int S = a.stages, BN = a.BN;
  const SmemLayout L = smem_layout(S, BN);
  uint8_t* sA = smem + L.a_off;
  uint8_t* sB = smem + L.b_off;
  float* xch = reinterpret_cast<float*>(smem + L.xch_off);
  float* red_v = reinterpret_cast<float*>(smem + L.red_off);
  int* red_i = reinterpret_cast<int*>(smem + L.red_off + 4 * 32 * 4);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t b_bytes = (uint32_t)BN * 128u;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiGroups * kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, (uint32_t)a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_begin();   // setup above overlaps the previous kernel; global reads/writes only from here
  const int ntiles = a.n_tiles_m * a.n_tiles_n;
  const int nunits = ntiles * a.splits;   // work unit = (tile, K split)

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once
      const uint64_t pol_x = policy_evict_last();   // activations: re-read by every m tile
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int t = u / a.splits, sk = u % a.splits;
        const int m = t / a.n_tiles_n, n = t % a.n_tiles_n;
        const int kb0 = sk * a.kb_per_split, kb1 = min(a.num_kb, kb0 + a.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kABytes + b_bytes);
          tma_load_2d_hint(sA + stage * kABytes, &tmA, &full[stage], kb * 64, m * 128, pol_w);
          tma_load_2d_hint(sB + stage * b_bytes, &tmB, &full[stage], kb * 64, n * BN, pol_x);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc = umma_idesc_bf16(128, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
        const int sk = u % a.splits;
        const int kb0 = sk * a.kb_per_split, kb1 = min(a.num_kb, kb0 + a.kb_per_split);
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * b_bytes);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            tc_mma_f16(d_tmem, umma_desc_sw128(a_addr + k * 32), umma_desc_sw128(b_addr + k * 32),
                       idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int tl = q * 32 + lane;      // tile-local feature (TMEM lane)
    const int gi = (warp - 2) >> 2;    // epilogue group
    const int et = (threadIdx.x - 64) & (kEpiThreads - 1);   // 0..127 thread id within the group
    float* gxch = xch + gi * (kXchBytes / 4);
    float* gred_v = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(red_v) + gi * kRedBytes);
    int* gred_i = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(red_i) + gi * kRedBytes);
    int it = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
      const int t = u / a.splits, sk = u % a.splits;
      const int m = t / a.n_tiles_n, n = t % a.n_tiles_n;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int nchunks = (BN + 31) / 32;
      for (int c = gi; c < nchunks; c += kEpiGroups) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
        tmem_ld_wait();
        const int row_base = n * BN + c * 32;
        const int ncol = min(32, BN - c * 32);
        epi_chunk<MODE>(a, v, m, tl, et, row_base, ncol, sk, gxch, gred_v, gred_i, 1 + gi);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (MODE == EPI_F32 && a.push && (et & 31) == 0) bulk_wait0();   // every pushed row has landed
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, (uint32_t)a.tmem_cols);
  }
}

// ------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a 256-feature x BN tile.
// CTA r loads weight rows [256p + 128r, +128) and activation rows [n*BN + r*BN/2, +BN/2) of each
// 64-deep k-block; the leader issues M=256 tcgen05.mma that read both CTAs' shared memory, so each
// SM receives 16 KB + BN*64 B per k-block instead of 16 KB + BN*128 B (operand delivery is the
// bottleneck of these skinny GEMMs).  Each CTA's TMEM holds its 128 features.
// ------------------------------------------------------------------------------------------
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;   // shared::cluster address of the leader's copy

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* m, uint64_t* leader_bar, int c0, int c1,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(leader_bar) & kPeerMask), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tc_mma_f16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_2sm_mc(uint64_t* bar, uint16_t mask = 3) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// 2SM TMA load multicast to the CTAs in `mask` (same smem offset in each); every destination's
// complete_tx goes to the barrier at leader_bar's offset in that destination's pair leader
__device__ __forceinline__ void tma_load_2d_2sm_mc(void* dst, const CUtensorMap* m, uint64_t* leader_bar, int c0,
                                                   int c1, uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5, %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(leader_bar) & kPeerMask), "r"(c0), "r"(c1), "h"(mask),
      "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// Work unit u of the CTA-pair kernel: tile t, K-slice sk, k-blocks [kb0, kb1); tail: one of the
// last-wave tiles' K-parts (GemmArgs::n_full)
struct Unit {
  int t, sk, kb0, kb1;
  bool tail;
};
__device__ __forceinline__ Unit unit_of(const GemmArgs& a, int u) {
  Unit r;
  const int nf = a.n_full * a.splits;
  if (u < nf) {
    r.t = u / a.splits;
    r.sk = u % a.splits;
    r.kb0 = r.sk * a.kb_per_split;
    r.kb1 = min(a.num_kb, r.kb0 + a.kb_per_split);
    r.tail = false;
  } else {
    const int v = u - nf;
    r.t = a.n_full + v / a.tail_split;
    r.sk = v % a.tail_split;
    r.kb0 = r.sk * a.kb_tail;
    r.kb1 = min(a.num_kb, r.kb0 + a.kb_tail);
    r.tail = true;
  }
  return r;
}

// Launched with clusters of 2*nc CTAs: nc CTA pairs compute the nc N-tiles of one 256-feature
// weight tile; pair 0 loads the weight halves once and multicasts them to every pair (the
// activation tiles differ per pair), which divides the L2->SM weight traffic by nc.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages, BN = a.BN, HB = BN / 2;
  const SmemLayout L = smem_layout(S, HB);
  uint8_t* sA = smem + L.a_off;
  uint8_t* sB = smem + L.b_off;
  float* xch = reinterpret_cast<float*>(smem + L.xch_off);
  float* red_v = reinterpret_cast<float*>(smem + L.red_off);
  int* red_i = reinterpret_cast<int*>(smem + L.red_off + 4 * 32 * 4);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int NC = a.nc;
  const int qp = (int)(rank >> 1);             // pair index in the cluster
  const uint32_t hr = rank & 1u;               // half of the pair
  const bool leader = hr == 0;
  const uint32_t b_bytes = (uint32_t)HB * 128u;
  // all CTAs of the cluster / the CTAs holding weight half hr / this pair
  const uint16_t mask_all = (uint16_t)((1u << (2 * NC)) - 1u);
  uint16_t mask_half = 0;
  for (int j = 0; j < NC; ++j) mask_half |= (uint16_t)(1u << (2 * j + hr));
  const uint16_t mask_pair = (uint16_t)(3u << (2 * qp));

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 2);         // one arrival per CTA of the pair (leader's carries the tx)
      mbar_init(&empty[s], NC);       // one MMA commit per pair (a stage holds multicast weights)
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiGroups * kEpiThreads);   // epilogue threads of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm(tmem_slot, (uint32_t)a.tmem_cols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_begin();   // setup above overlaps the previous kernel; global reads/writes only from here
  // cluster work unit = (256-feature tile p, N-tile group, K-split); pair qp takes N-tile
  // group * nc + qp (tiles past the activations read zeros and store nothing)
  // n_tiles_m counts 256-feature pairs here; mcx: n_groups counts groups of nc pairs
  const int ntiles = a.mcx ? a.n_groups * a.n_tiles_n : a.n_tiles_m * a.n_groups;
  // cluster tile t -> this pair's 256-feature tile p and activation tile n
  auto tile_pn = [&](int t, int& p, int& n) {
    if (a.mcx) {
      p = (t / a.n_tiles_n) * NC + qp;
      n = t % a.n_tiles_n;
    } else {
      p = t / a.n_groups;
      n = (t % a.n_groups) * NC + qp;
    }
  };
  const int nunits = a.n_full * a.splits + (ntiles - a.n_full) * a.tail_split;
  const int cl = blockIdx.x / (2 * NC), ncl = gridDim.x / (2 * NC);

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cl; u < nunits; u += ncl) {
        const Unit un = unit_of(a, u);
        int p, n;
        tile_pn(un.t, p, n);
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], 2 * (kABytes + b_bytes));
          else mbar_arrive_leader(&full[stage]);
          if (NC == 1 || a.mcx)
            tma_load_2d_2sm(sA + stage * kABytes, &tmA, &full[stage], kb * 64, p * 256 + (int)hr * 128, pol_w);
          else if (qp == 0)
            tma_load_2d_2sm_mc(sA + stage * kABytes, &tmA, &full[stage], kb * 64, p * 256 + (int)hr * 128, mask_half,
                               pol_w);
          if (NC == 1 || !a.mcx)
            tma_load_2d_2sm(sB + stage * b_bytes, &tmB, &full[stage], kb * 64, n * BN + (int)hr * HB, pol_x);
          else if (qp == 0)
            tma_load_2d_2sm_mc(sB + stage * b_bytes, &tmB, &full[stage], kb * 64, n * BN + (int)hr * HB, mask_half,
                               pol_x);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      const uint32_t idesc = umma_idesc_bf16(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cl; u < nunits; u += ncl, ++it) {
        const Unit un = unit_of(a, u);
        const int kb0 = un.kb0, kb1 = un.kb1;
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * b_bytes);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma_f16_2sm(d_tmem, umma_desc_sw128(a_addr + k * 32), umma_desc_sw128(b_addr + k * 32), idesc,
                           (kb > kb0 || k > 0) ? 1u : 0u);
          tc_commit_2sm_mc(&empty[stage], mask_all);   // every CTA's copy of the stage
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        tc_commit_2sm_mc(&tfull[acc], mask_pair);
      }
    }
  } else {
    const int q = warp & 3;
    const int tl = q * 32 + lane;
    const int gi = (warp - 2) >> 2;    // epilogue group
    const int et = (threadIdx.x - 64) & (kEpiThreads - 1);   // 0..127 thread id within the group
    float* gxch = xch + gi * (kXchBytes / 4);
    float* gred_v = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(red_v) + gi * kRedBytes);
    int* gred_i = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(red_i) + gi * kRedBytes);
    int it = 0;
    for (int u = cl; u < nunits; u += ncl, ++it) {
      const Unit un = unit_of(a, u);
      const int t = un.t, sk = un.sk;
      int p, n;
      tile_pn(t, p, n);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int nchunks = (BN + 31) / 32;
      if (p >= a.n_tiles_m) {   // mcx: a pair past the last 256-feature tile computed zeros
        tc_fence_before();
        mbar_arrive_leader(&tempty[acc]);
        continue;
      }
      if constexpr (MODE == EPI_SWIGLU) {
        if (un.tail) {
          // last-wave K-part: accumulator -> tail_buf[tail tile][part][pair][half][BN rows][128]
          // (coalesced over features), then the last part of (tile, pair, half) to finish sums the
          // parts in part order from L2 and runs the epilogue (fence / counter / last-arriver, no
          // CTA waits on another; a + b == b + a keeps any two-part order exact as well)
          const int ti = t - a.n_full;
          const size_t part_elems = (size_t)BN * 128;
          float* const tb = a.tail_buf + ((size_t)ti * a.tail_split * NC + qp) * 2 * part_elems + hr * part_elems;
          const size_t part_stride = (size_t)NC * 2 * part_elems;
          for (int c = gi; c < nchunks; c += kEpiGroups) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
            tmem_ld_wait();
            float* dst = tb + (size_t)sk * part_stride + (size_t)(c * 32) * 128 + tl;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c * 32 + j < BN) dst[(size_t)j * 128] = __uint_as_float(v[j]);
          }
          tc_fence_before();
          mbar_arrive_leader(&tempty[acc]);
          __threadfence();
          named_bar_sync(3, kEpiGroups * kEpiThreads);
          if (gi == 0 && et == 0) {
            int* cnt = a.tile_cnt + ((size_t)ti * NC + qp) * 2 + hr;
            const int prev = atomicAdd(cnt, 1);
            red_i[0] = prev == a.tail_split - 1;
            if (prev == a.tail_split - 1) *cnt = 0;   // ready for the next launch
          }
          named_bar_sync(3, kEpiGroups * kEpiThreads);
          if (red_i[0]) {
            __threadfence();
            for (int c = gi; c < nchunks; c += kEpiGroups) {
              // part by part (in order), all 32 rows' loads of a part in flight together
              float sv[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) sv[j] = 0.f;
              const float* src = tb + (size_t)(c * 32) * 128 + tl;
              const int nj = min(32, BN - c * 32);
#pragma unroll
              for (int s2 = 0; s2 < 8; ++s2) {
                if (s2 >= a.tail_split) break;
                float y[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) y[j] = j < nj ? __ldcg(src + (size_t)s2 * part_stride + (size_t)j * 128) : 0.f;
#pragma unroll
                for (int j = 0; j < 32; ++j) sv[j] += y[j];
              }
              uint32_t v[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(sv[j]);
              epi_chunk<MODE>(a, v, 2 * p + (int)hr, tl, et, n * BN + c * 32, min(32, BN - c * 32), 0, gxch, gred_v,
                              gred_i, 1 + gi);
            }
          }
          named_bar_sync(3, kEpiGroups * kEpiThreads);   // red_i[0] is rewritten by the next tail unit
          continue;
        }
      }
      for (int c = gi; c < nchunks; c += kEpiGroups) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
        tmem_ld_wait();
        const int row_base = n * BN + c * 32;
        const int ncol = min(32, BN - c * 32);
        epi_chunk<MODE>(a, v, 2 * p + (int)hr, tl, et, row_base, ncol, sk, gxch, gred_v, gred_i, 1 + gi);
      }
      tc_fence_before();
      mbar_arrive_leader(&tempty[acc]);
      if constexpr (MODE == EPI_F32) {
        if (a.resid && a.splits > 1) {
          // fused residual add of a K-split tile: the last split of (tile, CTA half) to finish sums
          // the partials from L2 in split order onto the residual stream (fence / counter /
          // last-arriver; no CTA waits on another); both epilogue groups' stores precede the count,
          // group 0 does the rest
          __threadfence();
          named_bar_sync(3, kEpiGroups * kEpiThreads);
        }
        if (a.resid && a.splits > 1 && gi == 0) {
          if (et == 0) {
            int* cnt = a.tile_cnt + ((size_t)t * NC + qp) * 2 + hr;
            const int prev = atomicAdd(cnt, 1);
            red_i[0] = prev == a.splits - 1;
            if (prev == a.splits - 1) *cnt = 0;   // ready for the next launch
          }
          named_bar_sync(1, kEpiThreads);
          if (red_i[0]) {
            __threadfence();
            // thread et: 4 consecutive features (float4) of rows et/32, et/32 + 4, ...; 4 rows per
            // thread in flight at once, every load of a batch issued before its stores
            const int f4 = (2 * p + (int)hr) * 128 + (et & 31) * 4;
            if (f4 < a.M) {
              const int r1 = min(a.R, (n + 1) * BN);
              constexpr int RB = 4;
              for (int r0 = n * BN + (et >> 5); r0 < r1; r0 += 4 * RB) {
                float4 acc_v[RB];
#pragma unroll
                for (int i = 0; i < RB; ++i) {
                  const int row = r0 + 4 * i;
                  acc_v[i] = row < r1 ? __ldcg(reinterpret_cast<const float4*>(a.resid + (size_t)row * a.ldo + f4))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                for (int s2 = 0; s2 < a.splits; ++s2) {
                  float4 y[RB];
#pragma unroll
                  for (int i = 0; i < RB; ++i) {
                    const int row = r0 + 4 * i;
                    y[i] = row < r1 ? __ldcg(reinterpret_cast<const float4*>(a.out_f32 + (size_t)s2 * a.split_stride +
                                                                              (size_t)row * a.ldo + f4))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                  }
#pragma unroll
                  for (int i = 0; i < RB; ++i) {
                    acc_v[i].x += y[i].x; acc_v[i].y += y[i].y; acc_v[i].z += y[i].z; acc_v[i].w += y[i].w;
                  }
                }
#pragma unroll
                for (int i = 0; i < RB; ++i)
                  if (r0 + 4 * i < r1) *reinterpret_cast<float4*>(a.resid + (size_t)(r0 + 4 * i) * a.ldo + f4) = acc_v[i];
              }
            }
          }
          named_bar_sync(1, kEpiThreads);   // red_i[0] is rewritten by the next tile
        }
      }
    }
    if (MODE == EPI_F32 && a.push && (et & 31) == 0) bulk_wait0();   // every pushed row has landed
  }
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, (uint32_t)a.tmem_cols);
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
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

thread_local int g_last_splits = 1;

template <int MODE>
cudaError_t launch_mode(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmArgs& a,
                        size_t smem, int grid, cudaStream_t st) {
  static PerDeviceOnce attr_set;   // the smem limit is a per-device attribute
  if (attr_set.first()) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) {
      attr_set.done.fetch_and(~(1ull << current_device()));
      return e;
    }
  }
  const cudaError_t le = launch_k(k_gemm<MODE>, dim3(grid), dim3(kThreads), smem, st, tmW, tmX, a);
  if (le != cudaSuccess) return le;
  return cudaGetLastError();
}

template <int MODE>
cudaError_t prep_mode2() {
  static PerDeviceOnce attr_set;   // the smem limit is a per-device attribute
  if (attr_set.first()) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm2<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) {
      attr_set.done.fetch_and(~(1ull << current_device()));
      return e;
    }
  }
  return cudaSuccess;
}

// clusters of `csize` CTAs that can be co-resident (cached per (mode, csize, smem))
template <int MODE>
int max_clusters2(int csize, size_t smem) {
  static std::map<std::pair<int, size_t>, int> cache;   // key: (device * 64 + csize, smem)
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(current_device() * 64 + csize, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize * 64, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_gemm2<MODE>, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = device_sms() / csize;
  }
  cache[key] = n;
  return n;
}

template <int MODE>
cudaError_t launch_mode2(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmArgs& a,
                         size_t smem, int grid, cudaStream_t st) {
  cudaError_t e = prep_mode2<MODE>();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2 * a.nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, k_gemm2<MODE>, tmW, tmX, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                  uint64_t row_stride) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {(row_stride ? row_stride : cols) * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int gemm_splits_last() { return g_last_splits; }

// Activation-row tile: the fewest <= 256-row tiles, rows rounded up to a multiple of 16
// (measured: 5 x 224 beats 6 x 176 for the 1056-row LM head; larger N per MMA instruction)
// The QKV projection runs with the fused RoPE epilogue (EPI_QKV, never K-split) when its pair
// tiles fit one wave of CTA pairs (one tile time; the fp32 path's K-split partials + RoPE kernel
// cost more: cfg5, 56 tiles, QKV + RoPE 2.0 -> 1.52 ms per step) or fill at least 1.5 waves
// (host-side estimate with one pair per two SMs); between the two the fp32 path's K split
// balances the waves better.
bool gemm_qkv_fused_ok(int M, int R) {
  const int g_num_sms = device_sms();
  const int bn = gemm_pick_bn(R);
  const int ntiles = ((M + 255) / 256) * ((R + bn - 1) / bn);
  const int nc = g_num_sms / 2;
  return ntiles <= nc || ntiles * 2 >= nc * 3;
}

int gemm_pick_bn(int R) {
  const int nt = (R + 255) / 256;
  int bn = (R + nt - 1) / nt;
  bn = (bn + 15) / 16 * 16;
  return std::max(16, std::min(256, bn));
}

namespace {
bool g_force_single = false;

cudaError_t gemm_launch_pair(int mode, const CUtensorMap& tmW, const void* X, GemmArgs a, cudaStream_t st,
                             int* launches) {
  const int HB = a.BN / 2;
  int ncols = 32;
  const int need = a.BN + (a.BN + 31) / 32 * 32;
  while (ncols < need) ncols *= 2;
  a.tmem_cols = ncols;
  const size_t budget = 227 * 1024 - 1024;
  int stages = 10;
  while (stages > 2 && smem_layout(stages, HB).total > budget) --stages;
  a.stages = stages;
  const size_t smem = smem_layout(stages, HB).total + 1024;
  CUtensorMap tmX;
  if (!make_tmap_2d(&tmX, X, (uint64_t)a.R, (uint64_t)a.K, (uint32_t)HB, (uint64_t)a.x_stride))
    return cudaErrorInvalidValue;
  const int n_pairs = (a.M + 255) / 256;
  // pairs per cluster sharing each weight tile through TMA multicast (SPECEDGE_GEMM_NC = 0: the
  // N-tiles of one 256-feature tile, up to 4 pairs).  Off by default: measured on cfg2 it cuts
  // the weights' L2 reads by 3x but the lock-stepped pairs and the cluster-of-6 occupancy
  // (22 clusters = 132 SMs) make the GEMM slower (profiles/README.md); the mainloop is bound by
  // operand delivery into shared memory, not by L2.
  static const int env_nc = getenv("SPECEDGE_GEMM_NC") ? atoi(getenv("SPECEDGE_GEMM_NC")) : 1;
  int nc = 1;
  if (env_nc > 0) nc = std::min(env_nc, 4);
  else if (a.n_tiles_n <= 4) nc = a.n_tiles_n;
  else if (a.n_tiles_n % 3 == 0) nc = 3;
  else if (a.n_tiles_n % 4 == 0) nc = 4;
  else if (a.n_tiles_n % 2 == 0) nc = 2;
  // SPECEDGE_GEMM_MCX=k: clusters of k pairs sharing the activation tile instead (pair 0
  // multicasts X; the weights are read per pair)
  static const int env_mcx = getenv("SPECEDGE_GEMM_MCX") ? atoi(getenv("SPECEDGE_GEMM_MCX")) : 0;
  a.mcx = (env_mcx > 1 && n_pairs >= 2 && !a.pair) ? 1 : 0;
  if (a.mcx) nc = std::min(std::min(env_mcx, 4), n_pairs);
  a.nc = nc;
  a.n_groups = a.mcx ? (n_pairs + nc - 1) / nc : (a.n_tiles_n + nc - 1) / nc;
  const int ntiles = a.mcx ? a.n_groups * a.n_tiles_n : n_pairs * a.n_groups;
  cudaError_t pe = cudaSuccess;
  int nclusters = 0;
  switch (mode) {
    case EPI_F32: pe = prep_mode2<EPI_F32>(); nclusters = max_clusters2<EPI_F32>(2 * nc, smem); break;
    case EPI_SWIGLU: pe = prep_mode2<EPI_SWIGLU>(); nclusters = max_clusters2<EPI_SWIGLU>(2 * nc, smem); break;
    case EPI_ARGMAX: pe = prep_mode2<EPI_ARGMAX>(); nclusters = max_clusters2<EPI_ARGMAX>(2 * nc, smem); break;
    case EPI_PQ1: pe = prep_mode2<EPI_PQ1>(); nclusters = max_clusters2<EPI_PQ1>(2 * nc, smem); break;
    case EPI_PQ2: pe = prep_mode2<EPI_PQ2>(); nclusters = max_clusters2<EPI_PQ2>(2 * nc, smem); break;
    case EPI_QKV: pe = prep_mode2<EPI_QKV>(); nclusters = max_clusters2<EPI_QKV>(2 * nc, smem); break;
    default: return cudaErrorInvalidValue;
  }
  if (pe != cudaSuccess) return pe;
  a.splits = 1;
  static const int env_max = getenv("SPECEDGE_MAX_SPLITS") ? atoi(getenv("SPECEDGE_MAX_SPLITS")) : 0;
  if (env_max > 0) a.max_splits = std::min(a.max_splits, env_max);
  const bool full_wave = a.unsplit_if_full && ntiles * 10 >= nclusters * 9 && ntiles <= nclusters;
  if (mode == EPI_F32 && !a.pair && a.max_splits > 1 && ntiles < nclusters * 3 / 2 && !full_wave) {
    int sp = (2 * nclusters + ntiles / 2) / ntiles;
    sp = std::min(sp, a.max_splits);
    while (sp > 1 && a.num_kb / sp < 8) --sp;
    a.splits = std::max(1, sp);
  }
  a.kb_per_split = (a.num_kb + a.splits - 1) / a.splits;
  g_last_splits = a.splits;
  // last-wave K split of the SwiGLU GEMM (stream-K style): the tail of ntiles % nclusters tiles
  // would otherwise leave the other clusters idle for a whole tile; split it into ts K-parts,
  // ts minimising the tail phase ceil(tail * ts / nclusters) / ts (in tile times) plus a
  // per-part cost of 0.04.  Off by default (SPECEDGE_TAIL_SPLIT=1 picks ts, =n forces it):
  // measured on cfg2 (ts = 3) gate/up 3.80 vs 3.38 ms per step — the parts alone would give 3.09,
  // but the last arriver's fixup (fence, counter, L2 reads of the parts, then the SwiGLU
  // epilogue: ~17 us on the critical path) costs more than the idle tail it removes
  // (profiles/README.md)
  a.n_full = ntiles;
  a.tail_split = 1;
  a.kb_tail = a.num_kb;
  static const int env_ts = getenv("SPECEDGE_TAIL_SPLIT") ? atoi(getenv("SPECEDGE_TAIL_SPLIT")) : -1;
  if (mode == EPI_SWIGLU && a.tail_buf && a.tile_cnt && env_ts > 0 && ntiles > nclusters) {
    const int tail = ntiles % nclusters;
    int best = 1;
    double best_cost = 1.0;
    for (int ts = 2; ts <= 8 && tail > 0; ++ts) {
      if (a.num_kb / ts < 8) break;
      if ((size_t)tail * ts * nc * 2 * a.BN * 128 * 4 > a.tail_cap) break;
      const double cost = (double)((tail * ts + nclusters - 1) / nclusters) / ts + 0.04 * ts;
      if (env_ts > 1 ? ts == env_ts : cost < best_cost) { best = ts; best_cost = cost; }
    }
    if (best > 1) {
      a.n_full = ntiles - tail;
      a.tail_split = best;
      a.kb_tail = (a.num_kb + best - 1) / best;
    }
  }
  GemmArgs b = a;
  b.n_tiles_m = n_pairs;      // the kernel iterates 256-feature pairs
  const int nunits_h = a.n_full * a.splits + (ntiles - a.n_full) * a.tail_split;
  const int grid = 2 * nc * std::min(nunits_h, nclusters);
  if (launches) ++*launches;
  switch (mode) {
    case EPI_F32: return launch_mode2<EPI_F32>(tmW, tmX, b, smem, grid, st);
    case EPI_SWIGLU: return launch_mode2<EPI_SWIGLU>(tmW, tmX, b, smem, grid, st);
    case EPI_ARGMAX: return launch_mode2<EPI_ARGMAX>(tmW, tmX, b, smem, grid, st);
    case EPI_PQ1: return launch_mode2<EPI_PQ1>(tmW, tmX, b, smem, grid, st);
    case EPI_PQ2: return launch_mode2<EPI_PQ2>(tmW, tmX, b, smem, grid, st);
    case EPI_QKV: return launch_mode2<EPI_QKV>(tmW, tmX, b, smem, grid, st);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

void gemm_force_single(bool on) { g_force_single = on; }

cudaError_t gemm_launch(int mode, const CUtensorMap& tmW, const void* X, GemmArgs a,
                        cudaStream_t st, int* launches) {
  const int g_num_sms = device_sms();
  a.BN = a.bn_override > 0 ? a.bn_override : gemm_pick_bn(a.R);
  a.n_tiles_n = (a.R + a.BN - 1) / a.BN;
  a.n_tiles_m = (a.M + 127) / 128;
  a.ntm128 = a.n_tiles_m;
  a.num_kb = (a.K + 63) / 64;
  // CTA pairs whenever the weight side has >= 2 128-row tiles (the pair needs BN/2 rows per CTA
  // aligned to 8 rows: BN is a multiple of 16)
  static const bool env_single = getenv("SPECEDGE_GEMM_SINGLE") && getenv("SPECEDGE_GEMM_SINGLE")[0] == '1';
  const bool pair_mode = !g_force_single && !env_single && a.n_tiles_m >= 2;
  if (pair_mode) return gemm_launch_pair(mode, tmW, X, a, st, launches);
  int ncols = 32;
  const int need = a.BN + (a.BN + 31) / 32 * 32;
  while (ncols < need) ncols *= 2;
  a.tmem_cols = ncols;
  const size_t budget = 227 * 1024 - 1024;
  int stages = 8;
  while (stages > 2 && smem_layout(stages, a.BN).total > budget) --stages;
  a.stages = stages;
  const size_t smem = smem_layout(stages, a.BN).total + 1024;
  CUtensorMap tmX;
  if (!make_tmap_2d(&tmX, X, (uint64_t)a.R, (uint64_t)a.K, (uint32_t)a.BN, (uint64_t)a.x_stride))
    return cudaErrorInvalidValue;
  const int ntiles = a.n_tiles_m * a.n_tiles_n;
  // K-split (EPI_F32 only, caller provides max_splits slices of split_stride floats): give every
  // CTA >= 2 units so the epilogue of one overlaps the MMAs of the next, and fill the SMs.
  a.splits = 1;
  // (the single-CTA kernel has no split fixup: a fused residual add runs unsplit here)
  if (mode == EPI_F32 && !a.pair && !a.resid && a.max_splits > 1 && ntiles < g_num_sms * 3 / 2) {
    int sp = (2 * g_num_sms + ntiles / 2) / ntiles;
    sp = std::min(sp, a.max_splits);
    while (sp > 1 && a.num_kb / sp < 8) --sp;
    a.splits = std::max(1, sp);
  }
  a.kb_per_split = (a.num_kb + a.splits - 1) / a.splits;
  g_last_splits = a.splits;
  const int grid = std::min(ntiles * a.splits, g_num_sms);
  if (launches) ++*launches;
  switch (mode) {
    case EPI_F32: return launch_mode<EPI_F32>(tmW, tmX, a, smem, grid, st);
    case EPI_SWIGLU: return launch_mode<EPI_SWIGLU>(tmW, tmX, a, smem, grid, st);
    case EPI_ARGMAX: return launch_mode<EPI_ARGMAX>(tmW, tmX, a, smem, grid, st);
    case EPI_PQ1: return launch_mode<EPI_PQ1>(tmW, tmX, a, smem, grid, st);
    case EPI_PQ2: return launch_mode<EPI_PQ2>(tmW, tmX, a, smem, grid, st);
    case EPI_QKV: return launch_mode<EPI_QKV>(tmW, tmX, a, smem, grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace se
