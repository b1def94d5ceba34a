// Tree-masked paged split-KV attention ("custom attention masking
// for each token sequence in the batch ... without cross-sequence interference").
//
// Work item = (request r, kv head g, split sp).  Its query rows are the request's S slots x the
// G query heads that share kv head g (row i = s*G + j).  Keys: the cached prefix [0, L_r) read
// from 64-token pages through the block table (split sp takes a contiguous page range), plus —
// in the last split — the S tree slots of this step from the tree K/V scratch, where slot s sees
// slot t iff t == 0 (root) or node t-1 is an ancestor-or-self of node s-1 (uint64 bitmask).
// Scores fp32, online softmax in the log2 domain; P enters the PV product as fp16 (q, k, v and the
// KV cache are fp16, DESIGN.md R-precision; P in bf16 would give ~1.5e-3 relative error).
// QK^T and PV use mma.sync m16n8k16 (16-row granularity suits the ragged S*G row counts);
// K/V tiles are staged into XOR-swizzled shared memory with cp.async, double-buffered.
// Partials (o, m, l) per split are merged by k_attn_combine.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cstdlib>

namespace se {

namespace {

constexpr int kMaxWarps = 12;   // 384 threads -> up to 170 registers/thread

__device__ __forceinline__ int swz(int row, int chunk, int nchunks) {
  const int m = nchunks >= 8 ? 7 : nchunks - 1;
  return chunk ^ (row & m);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_f16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Load a [64 keys][HD] fp16 tile (rows beyond `valid` zero-filled) into swizzled smem.
template <int HD>
__device__ __forceinline__ void load_tile(f16* dst, const f16* src, int valid, int tid, int nthreads) {
  constexpr int NCH = HD / 8;
  for (int i = tid; i < 64 * NCH; i += nthreads) {
    const int r = i / NCH, c = i % NCH;
    const bool ok = r < valid;
    const f16* s = ok ? src + (size_t)r * HD + c * 8 : src;
    cp_async16(dst + r * HD + swz(r, c, NCH) * 8, s, ok);
  }
}

template <int HD>
__global__ void __launch_bounds__(kMaxWarps * 32)
    k_tree_attention(const __grid_constant__ AttnArgs a) {
  pdl_begin();
  constexpr int NCH = HD / 8;      // 16-byte chunks per row
  constexpr int KS = HD / 16;      // k16 steps over head dim
  constexpr int NT = HD / 8;       // n8 tiles over head dim
  extern __shared__ __align__(128) uint8_t smem_raw[];
  f16* sQ = reinterpret_cast<f16*>(smem_raw);                     // [max_rows_pad][HD]
  const int rows_pad = (a.max_rows + 15) / 16 * 16;
  f16* sK = sQ + (size_t)rows_pad * HD;                           // [2][64][HD]
  f16* sV = sK + 2 * 64 * HD;                                     // [2][64][HD]
  uint64_t* sAnc = reinterpret_cast<uint64_t*>(sV + 2 * 64 * HD); // [max_S]

  const int r = blockIdx.x / a.KV, g = blockIdx.x % a.KV, sp = blockIdx.y;
  const int tid = threadIdx.x, nthreads = blockDim.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = nthreads >> 5;
  const int G = a.G;
  const int S = min(a.req_S[r], a.max_rows / G);
  const int rows = S * G;
  const int L = a.req_L[r];
  const int row0 = a.req_row0[r];
  const int h = a.req_h[r];

  // page range of this split; the tree block goes to the last split
  const int npages = (L + 63) / 64;
  const int p_begin = sp * a.pages_per_split;
  const int p_end = min(npages, p_begin + a.pages_per_split);
  const bool has_tree = sp == a.n_splits - 1;
  const int n_prefix_tiles = max(0, p_end - p_begin);
  const int n_tree_tiles = has_tree ? (S + 63) / 64 : 0;
  const int ntiles = n_prefix_tiles + n_tree_tiles;

  // Q rows (s, j) -> smem, swizzled; anc masks
  for (int i = tid; i < rows_pad * NCH; i += nthreads) {
    const int qr = i / NCH, c = i % NCH;
    const int s = qr / G, j = qr % G;
    const bool ok = qr < rows;
    const f16* src = ok ? a.Q + (size_t)(row0 + s) * (a.H * HD) + (size_t)(g * G + j) * HD + c * 8 : a.Q;
    cp_async16(sQ + qr * HD + swz(qr, c, NCH) * 8, src, ok);
  }
  for (int s = tid; s < S; s += nthreads) sAnc[s] = a.row_anc[row0 + s];
  cp_async_commit();

  auto tile_src = [&](int t, const f16*& ks, const f16*& vs, int& valid, int& key0) {
    if (t < n_prefix_tiles) {
      const int p = p_begin + t;
      const int page = a.block_table[(size_t)h * a.max_pages_per_seq + p];
      const size_t base = ((((size_t)a.layer * a.num_pages + page) * 2) * a.KV + g) * 64 * HD;
      ks = a.pool + base;
      vs = a.pool + base + (size_t)a.KV * 64 * HD;
      valid = min(64, L - p * 64);
      key0 = -1;
    } else {
      const int tt = t - n_prefix_tiles;
      const size_t kb = (((size_t)a.layer * 2 + 0) * a.KV + g) * a.R_cap;
      const size_t vb = (((size_t)a.layer * 2 + 1) * a.KV + g) * a.R_cap;
      ks = a.tree_kv + (kb + row0 + tt * 64) * HD;
      vs = a.tree_kv + (vb + row0 + tt * 64) * HD;
      valid = min(64, S - tt * 64);
      key0 = tt * 64;   // tree slot index of key 0
    }
  };

  if (ntiles > 0) {
    const f16 *ks, *vs;
    int valid, key0;
    tile_src(0, ks, vs, valid, key0);
    load_tile<HD>(sK, ks, valid, tid, nthreads);
    load_tile<HD>(sV, vs, valid, tid, nthreads);
  }
  cp_async_commit();

  const float sl2 = a.scale_log2;
  const int n_row_tiles = (rows + 15) / 16;
  // each warp owns row tiles warp, warp + nwarps, ... ; all tiles of a group share one K/V pass
  const int n_groups = max(1, (n_row_tiles + nwarps - 1) / nwarps);

  for (int grp = 0; grp < n_groups; ++grp) {
    const int rt = grp * nwarps + warp;
    const bool active = rt < n_row_tiles;
    float o[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    uint32_t qf[KS][4];
    // rows this thread's accumulators refer to
    const int qr0 = rt * 16 + (lane >> 2), qr1 = qr0 + 8;
    const int s0 = qr0 / G, s1 = qr1 / G;
    uint64_t anc0 = 0, anc1 = 0;

    if (grp > 0) {
      // restart the K/V stream for the next row group
      __syncthreads();
      if (ntiles > 0) {
        const f16 *ks, *vs;
        int valid, key0;
        tile_src(0, ks, vs, valid, key0);
        load_tile<HD>(sK, ks, valid, tid, nthreads);
        load_tile<HD>(sV, vs, valid, tid, nthreads);
      }
      cp_async_commit();
    }

    for (int t = 0; t < ntiles; ++t) {
      const int buf = t & 1;
      if (t + 1 < ntiles) {
        const f16 *ks, *vs;
        int valid, key0;
        tile_src(t + 1, ks, vs, valid, key0);
        load_tile<HD>(sK + (buf ^ 1) * 64 * HD, ks, valid, tid, nthreads);
        load_tile<HD>(sV + (buf ^ 1) * 64 * HD, vs, valid, tid, nthreads);
        cp_async_commit();
        cp_async_wait_1();
      } else {
        cp_async_wait_all();
      }
      __syncthreads();
      if (t == 0 && active) {
        // Q fragments (A operand, row-major): matrices (rows 0-7,k0-7),(8-15,k0-7),(0-7,k8-15),(8-15,k8-15)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int mat = lane >> 3, rr = lane & 7;
          const int qr = rt * 16 + rr + (mat & 1) * 8;
          const int ch = ks * 2 + (mat >> 1);
          ldsm_x4(smem_u32(sQ + qr * HD + swz(qr, ch, NCH) * 8), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
        }
        if (s0 < S) anc0 = sAnc[s0];
        if (s1 < S) anc1 = sAnc[s1];
      }
      if (active) {
        const f16* cK = sK + buf * 64 * HD;
        const f16* cV = sV + buf * 64 * HD;
        const f16 *ks_, *vs_;
        int valid, key0;
        tile_src(t, ks_, vs_, valid, key0);
        // S = Q K^T : 16 rows x 64 keys
        float sc[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
          for (int np = 0; np < 4; ++np) {   // pairs of n8 key tiles
            const int mat = lane >> 3, rr = lane & 7;
            const int kr = np * 16 + rr + (mat >> 1) * 8;
            const int ch = ks * 2 + (mat & 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4(smem_u32(cK + kr * HD + swz(kr, ch, NCH) * 8), b0, b1, b2, b3);
            mma_f16(sc[np * 2], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b0, b1);
            mma_f16(sc[np * 2 + 1], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b2, b3);
          }
        }
        // mask + scale (log2 domain)
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = nt * 8 + (lane & 3) * 2 + (e & 1);
            const int hr = e >> 1;
            const int srow = hr ? s1 : s0;
            bool ok = key < valid && srow < S;
            if (ok && key0 >= 0) {
              const int slot = key0 + key;   // tree slot of this key
              const uint64_t an = hr ? anc1 : anc0;
              ok = slot == 0 || (srow > 0 && ((an >> (slot - 1)) & 1ull));
            }
            const float v = ok ? sc[nt][e] * sl2 : -INFINITY;
            sc[nt][e] = v;
            mx[hr] = fmaxf(mx[hr], v);
          }
        }
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffff, mx[hr], 1));
          mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffff, mx[hr], 2));
        }
        float alpha[2], base[2], rs[2] = {0.f, 0.f};
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          const float mn = fmaxf(mrow[hr], mx[hr]);
          base[hr] = mn == -INFINITY ? 0.f : mn;
          alpha[hr] = exp2f(mrow[hr] - base[hr]);
          mrow[hr] = mn;
        }
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float p = exp2f(sc[nt][e] - base[e >> 1]);
            sc[nt][e] = p;
            rs[e >> 1] += p;
          }
        }
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          rs[hr] += __shfl_xor_sync(0xffffffff, rs[hr], 1);
          rs[hr] += __shfl_xor_sync(0xffffffff, rs[hr], 2);
          lrow[hr] = lrow[hr] * alpha[hr] + rs[hr];
        }
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          o[i][0] *= alpha[0];
          o[i][1] *= alpha[0];
          o[i][2] *= alpha[1];
          o[i][3] *= alpha[1];
        }
        // O += P V (P fp16)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float* c0 = sc[2 * kk];
          const float* c1 = sc[2 * kk + 1];
          // A regs: a0=(row,k0-1) a1=(row+8,k0-1) a2=(row,k8-9) a3=(row+8,k8-9)
          const uint32_t a0 = pack_f16(c0[0], c0[1]), a1 = pack_f16(c0[2], c0[3]);
          const uint32_t a2 = pack_f16(c1[0], c1[1]), a3 = pack_f16(c1[2], c1[3]);
#pragma unroll
          for (int np = 0; np < NT / 2; ++np) {   // pairs of n8 dim tiles
            const int mat = lane >> 3, rr = lane & 7;
            const int kr = kk * 16 + rr + (mat & 1) * 8;
            const int ch = np * 2 + (mat >> 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(smem_u32(cV + kr * HD + swz(kr, ch, NCH) * 8), b0, b1, b2, b3);
            mma_f16(o[np * 2], a0, a1, a2, a3, b0, b1);
            mma_f16(o[np * 2 + 1], a0, a1, a2, a3, b2, b3);
          }
        }
      }
      __syncthreads();   // buffer `buf` is refilled at iteration t+2 (issued at t+1)
    }

    // write partials for this warp's 16 rows
    if (active) {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int qr = hr ? qr1 : qr0;
        if (qr >= rows) continue;
        const int s = qr / G, j = qr % G;
        const size_t rh = (size_t)(row0 + s) * a.H + (size_t)g * G + j;
        const size_t pb = (size_t)sp * a.R * a.H + rh;
        float* op = a.opart + pb * HD;
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          const int d = i * 8 + (lane & 3) * 2;
          *reinterpret_cast<float2*>(op + d) = make_float2(o[i][hr * 2], o[i][hr * 2 + 1]);
        }
        if ((lane & 3) == 0) {
          a.mpart[pb] = mrow[hr];
          a.lpart[pb] = lrow[hr];
        }
      }
    }
  }
  cp_async_wait_all();
}

// Merge split partials: o = sum_sp 2^(m_sp - m) o_sp / sum_sp 2^(m_sp - m) l_sp.
// One warp per (row, head); lanes own 4 consecutive head-dim elements (float4).
__global__ void k_attn_combine(const __grid_constant__ AttnArgs a, bf16* __restrict__ O,
                               float* __restrict__ O_f32) {
  pdl_begin();
  // one warp per (row, kv head g): the chunk count is looked up once for the G query heads of
  // the group; every partial a head needs is loaded in one round, two heads in flight
  const int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // row * KV + g
  const int lane = threadIdx.x & 31;
  if (item >= a.R * a.KV) return;
  const int row = item / a.KV, g = item % a.KV;
  const int hd = a.hd;
  const size_t stride = (size_t)a.R * a.H;
  int ns = a.n_splits;
  if (a.per_req == 1) {
    const int r = a.row_req ? a.row_req[row] : 0;
    const int npages = (a.req_L[r] + 63) / 64;
    ns = max(1, (npages + a.pages_per_split - 1) / a.pages_per_split);
    if (ns == 1) return;   // written final by the attention kernel
  } else if (a.per_req == 2) {
    // balanced tcgen05 attention: the kernel recorded the chunk count of every (r, g)
    const int r = a.row_req ? a.row_req[row] : 0;
    ns = a.nch_tab[r * a.KV + g];
    if (ns == 1) return;
  }
  constexpr int kCombineMax = 8;
  const int d = lane * 4;
  const bool has_d = d < hd;
#pragma unroll 2
  for (int j = 0; j < a.G; ++j) {
    const size_t rh = (size_t)row * a.H + (size_t)g * a.G + j;
    float mv[kCombineMax], lv[kCombineMax];
    float4 ov[kCombineMax];
#pragma unroll
    for (int sp = 0; sp < kCombineMax; ++sp) {
      const bool on = sp < ns;
      mv[sp] = on ? a.mpart[sp * stride + rh] : -INFINITY;
      lv[sp] = on ? a.lpart[sp * stride + rh] : 0.f;
      ov[sp] = (on && has_d) ? *reinterpret_cast<const float4*>(a.opart + (sp * stride + rh) * hd + d)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float m = -INFINITY;
#pragma unroll
    for (int sp = 0; sp < kCombineMax; ++sp) m = fmaxf(m, mv[sp]);
    const float mb = m == -INFINITY ? 0.f : m;
    float l = 0.f;
    float w[kCombineMax];
#pragma unroll
    for (int sp = 0; sp < kCombineMax; ++sp) {
      w[sp] = mv[sp] == -INFINITY ? 0.f : exp2f(mv[sp] - mb);
      l += w[sp] * lv[sp];
    }
    const float inv = l > 0.f ? 1.0f / l : 0.f;
    if (!has_d) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int sp = 0; sp < kCombineMax; ++sp) {
      const float ww = w[sp] * inv;
      if (ww != 0.f) {   // skipped partials (no visible key, or sp >= ns) may hold stale values
        acc.x += ww * ov[sp].x;
        acc.y += ww * ov[sp].y;
        acc.z += ww * ov[sp].z;
        acc.w += ww * ov[sp].w;
      }
    }
    if (O) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(acc.x, acc.y), p1 = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&p0);
      u.y = *reinterpret_cast<uint32_t*>(&p1);
      *reinterpret_cast<uint2*>(O + rh * hd + d) = u;
    }
    if (O_f32) *reinterpret_cast<float4*>(O_f32 + rh * hd + d) = acc;
  }
}

template <int HD>
cudaError_t launch_hd(const AttnArgs& a, int B, cudaStream_t st) {
  const int rows_pad = (a.max_rows + 15) / 16 * 16;
  const int nwarps = std::max(1, std::min(kMaxWarps, rows_pad / 16));
  const int max_S = a.max_rows / a.G;
  const size_t smem = (size_t)rows_pad * HD * 2 + 4 * 64 * HD * 2 + (size_t)max_S * 8 + 16;
  static size_t attr[kMaxDevices] = {};   // per-device attribute
  const int dev = current_device();
  if (smem > attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_tree_attention<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max(smem, (size_t)48 * 1024));
    if (e != cudaSuccess) return e;
    attr[dev] = std::max(smem, (size_t)48 * 1024);
  }
  dim3 grid(B * a.KV, a.n_splits);
  {
    cudaError_t le = launch_k(k_tree_attention<HD>, grid, dim3(nwarps * 32), smem, st, a);
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}

}  // namespace

// tcgen05 kernel: one CTA per SM (512 TMEM columns).  Short contexts: split only when (request,
// kv head) items leave most SMs idle.  Long contexts (>= 64 pages): cut every request's pages
// into chunks of P pages so that the chunks fill about `waves` rounds of the 148 SMs; the
// hardware block scheduler then balances ragged context lengths (cfg5: 192-320 pages per request
// would otherwise leave the longest CTA running 1.25x the mean with 20 SMs idle).
int attn_pick_chunk_tc(int B, int KV, int max_pages) {
  static const int env_p = getenv("SPECEDGE_ATTN_CHUNK") ? atoi(getenv("SPECEDGE_ATTN_CHUNK")) : 0;
  static const int waves = getenv("SPECEDGE_ATTN_WAVES") ? std::max(1, atoi(getenv("SPECEDGE_ATTN_WAVES"))) : 4;
  max_pages = std::max(1, max_pages);
  if (env_p > 0) return std::max(env_p, (max_pages + 7) / 8);
  const int items = std::max(1, B * KV);
  if (max_pages < 64) {
    int ns = (148 + items / 2) / items;
    ns = std::min(ns, 8);
    ns = std::min(ns, std::max(1, (max_pages + 1) / 2));
    ns = std::max(1, ns);
    return (max_pages + ns - 1) / ns;
  }
  const long long want = ((long long)items * max_pages + 148LL * waves - 1) / (148LL * waves);
  return (int)std::min<long long>(max_pages, std::max<long long>({want, (max_pages + 7) / 8, 8}));
}

int attn_pick_splits(int B, int KV, int max_pages) {
  const int items = std::max(1, B * KV);
  int ns = (2 * 148 + items - 1) / items;
  ns = std::min(ns, 16);
  ns = std::min(ns, std::max(1, max_pages));
  return std::max(1, ns);
}

cudaError_t attention_launch(const AttnArgs& a, int B, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  switch (a.hd) {
    case 16: return launch_hd<16>(a, B, st);
    case 32: return launch_hd<32>(a, B, st);
    case 64: return launch_hd<64>(a, B, st);
    case 128: return launch_hd<128>(a, B, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t attn_combine_launch(const AttnArgs& a, bf16* O, float* O_f32, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  {
    cudaError_t le = launch_k(k_attn_combine, dim3((a.R * a.KV + 7) / 8), dim3(256), 0, st, a, O, O_f32);
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}

}  // namespace se
