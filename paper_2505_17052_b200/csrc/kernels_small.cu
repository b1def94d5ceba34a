// Integer / bandwidth kernels of the verify step:
//   K1  tree prep     (S:111 tree invariants, amb. A3-A5, A18)
//   K2  embedding gather (a2)
//   K3  RMSNorm       (a3, amb. A13)
//   K9b LM-head second stage: argmax over per-tile partials (a9, ties -> lowest id)
//   K10 accept walk   (a10; "returns both the verified tokens and one additional token")
//   K11 KV commit     (a11; amb. A19) + length finalize
//   K12 Philox weight init, K13 synthetic KV fill
#include "common.cuh"
#include "internal.h"

namespace se {
#define CK_RET(x)                 \
  do {                            \
    cudaError_t _e = (x);         \
    if (_e != cudaSuccess) return _e; \
  } while (0)


namespace {

// ------------------------------------------------------------------------------------ K1 prep
// One CTA (64 threads) per request.  Thread i owns node i (and i+64.. when N > 64 so every row
// is still written for oversize trees, which are flagged E_TREE_SIZE).
__global__ void k_prep(const __grid_constant__ PrepArgs p) {
  pdl_begin();
  const int r = blockIdx.x, i0 = threadIdx.x;
  __shared__ int s_flags[8];
  __shared__ int s_depth_max;
  __shared__ int s_parent[kMaxNodes];
  __shared__ int s_token[kMaxNodes];
  const int n0 = p.node_offset[r];
  const int N = p.node_offset[r + 1] - n0;
  const int row0 = n0 + r;
  if (i0 < 8) s_flags[i0] = 0;
  if (i0 == 0) s_depth_max = 0;
  for (int i = i0; i < min(N, kMaxNodes); i += blockDim.x) {
    s_parent[i] = p.parent[n0 + i];
    s_token[i] = p.token[n0 + i];
  }
  __syncthreads();

  // handle: in range, allocated, not used by an earlier request of this batch
  const int h = p.kv[r];
  bool handle_ok = h >= 0 && h < p.max_handles && p.capacity[h] > 0;
  if (handle_ok) {
    for (int j = i0; j < r; j += blockDim.x)
      if (p.kv[j] == h) atomicOr(&s_flags[0], 1);
  }
  const bool size_ok = N >= 0 && N <= kMaxNodes && N <= p.max_nodes;
  // per-node checks (only meaningful when the size is ok)
  if (size_ok) {
    for (int i = i0; i < N; i += blockDim.x) {
      const int par = s_parent[i];
      if (!(par == -1 || (par >= 0 && par < i))) atomicOr(&s_flags[1], 1);
      const int tk = s_token[i];
      if (tk < 0 || tk >= p.V) atomicOr(&s_flags[2], 1);
      for (int j = 0; j < i; ++j)
        if (s_parent[j] == par && s_token[j] == tk) atomicOr(&s_flags[3], 1);
    }
  }
  __syncthreads();
  const bool tree_ok = size_ok && s_flags[1] == 0;
  const int root = p.root_token[r];

  // depth / ancestor mask by walking the parent chain (<= 64 steps)
  __shared__ int s_depth[kMaxNodes];
  for (int i = i0; i < N; i += blockDim.x) {
    int depth = 1;
    uint64_t anc = 0;
    if (tree_ok) {
      anc = 1ull << i;
      int c = s_parent[i];
      while (c >= 0) {
        anc |= 1ull << c;
        ++depth;
        c = s_parent[c];
      }
      atomicMax(&s_depth_max, depth);
    }
    if (i < kMaxNodes) s_depth[i] = depth;
    const int tk = i < kMaxNodes ? s_token[i] : p.token[n0 + i];
    p.row_tok[row0 + 1 + i] = (tk >= 0 && tk < p.V) ? tk : 0;
    p.row_anc[row0 + 1 + i] = anc;
    p.row_req[row0 + 1 + i] = r;
    p.row_slot[row0 + 1 + i] = i + 1;
  }
  __syncthreads();

  const bool h_ok = handle_ok && s_flags[0] == 0;
  const int L = h_ok ? p.cache_len[h] : 0;
  for (int i = i0; i < N; i += blockDim.x) p.row_pos[row0 + 1 + i] = L + (i < kMaxNodes ? s_depth[i] : 1);
  if (i0 == 0) {
    int st = SPECEDGE_REQ_OK;
    if (!h_ok) st = SPECEDGE_REQ_E_HANDLE;
    else if (!size_ok) st = SPECEDGE_REQ_E_TREE_SIZE;
    else if (s_flags[1]) st = SPECEDGE_REQ_E_TREE;
    else if (s_flags[2] || root < 0 || root >= p.V) st = SPECEDGE_REQ_E_TOKEN;
    else if (s_flags[3]) st = SPECEDGE_REQ_E_DUP_SIBLING;
    else if (p.context_len[r] != L + 1 || p.context_len[r] > p.max_context_len || L + s_depth_max >= p.max_position)
      st = SPECEDGE_REQ_E_CONTEXT;
    else if (L + s_depth_max + 1 > p.capacity[h]) st = SPECEDGE_REQ_E_KV_CAPACITY;
    p.status[r] = st;
    p.req_L[r] = L;
    p.req_h[r] = h_ok ? h : 0;
    p.req_row0[r] = row0;
    p.req_S[r] = N + 1;
    p.row_tok[row0] = (root >= 0 && root < p.V) ? root : 0;
    p.row_pos[row0] = L;
    p.row_anc[row0] = 0;
    p.row_req[row0] = r;
    p.row_slot[row0] = 0;
  }
}

// ------------------------------------------------------------------------------- K2 embedding
// X (fp32 residual stream) = E[token] (bf16 values, exact in fp32)
__global__ void k_embed(const bf16* __restrict__ E, const int* __restrict__ row_tok, float* __restrict__ X, int d) {
  pdl_begin();
  const int row = blockIdx.x;
  const int tok = row_tok[row];
  const uint4* src = reinterpret_cast<const uint4*>(E + (size_t)tok * d);
  float4* dst = reinterpret_cast<float4*>(X + (size_t)row * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    const uint4 u = src[i];
    dst[2 * i] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                             __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
    dst[2 * i + 1] = make_float4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xFFFF0000u),
                                 __uint_as_float(u.w << 16), __uint_as_float(u.w & 0xFFFF0000u));
  }
}

// --------------------------------------------------------------------------------- K3 RMSNorm
// Residual add + RMSNorm (amb. A13): x = X + Y[0] + ... + Y[nY-1] (the O-proj / down GEMM's K-split
// partials, summed in this fixed order), X = x (fp32 residual stream), out = bf16(x * rsqrt(mean(x^2)
// + eps) * g).  split = 1 (final norm feeding the LM head): y is written as two bf16 rows, hi =
// bf16(y) at out row 2r and lo = bf16(y - hi) at row 2r+1, so hi + lo carries y to ~2^-17.
// ys (NEXT-F4, tensor parallel): partial s of this rank's rows at ys.p[s] (a peer's memory over
// NVLink for s != own rank) instead of Y + s * y_stride; summed in the same fixed order.
// NY < 0 (more than 4 partials, tensor parallel at 5-8 ranks): -NY partials summed one at a time
// in the same fixed order (no register prefetch of all of them).
template <int NY>
__global__ void __launch_bounds__(1024) k_rmsnorm(float* __restrict__ X, const float* __restrict__ Y, size_t y_stride,
                                                  const bf16* __restrict__ g, bf16* __restrict__ out, int d, float eps,
                                                  int split, const RmsSrc ys) {
  pdl_begin();
  // blockDim.x = d / 16 rounded up to whole warps, T threads: thread t owns the float4 groups
  // t + T*k (k < 4), i.e. elements [4(t + Tk), 4(t + Tk) + 4), kept in registers across passes —
  // every warp-wide load / store covers 512 contiguous bytes; groups past d hold zeros and neither
  // load nor store, so the full-mask warp reductions below always run on complete warps
  const int row = blockIdx.x;
  const int T = blockDim.x;
  const int t = threadIdx.x;
  float* x = X + (size_t)row * d;
  __shared__ float red[32];
  float4 xv[4];
  bool own[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    own[k] = 4 * (t + T * k) < d;
    xv[k] = own[k] ? *reinterpret_cast<const float4*>(x + 4 * (t + T * k)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if constexpr (NY > 0) {
    float4 yv[NY][4];
#pragma unroll
    for (int s = 0; s < NY; ++s)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!own[k]) {
          yv[s][k] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else if (NY == 1 && ys.mc) {   // NVLS: the sum over all ranks' partials, reduced in the switch
          const float* pm = ys.mc + (size_t)row * d + 4 * (t + T * k);
          float4 v;
          asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "l"(pm)
                       : "memory");
          yv[s][k] = v;
        } else {
          yv[s][k] = __ldcs(reinterpret_cast<const float4*>((ys.p[0] ? ys.p[s] : Y + s * y_stride) + (size_t)row * d +
                                                            4 * (t + T * k)));
        }
      }
#pragma unroll
    for (int s = 0; s < NY; ++s)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        xv[k].x += yv[s][k].x; xv[k].y += yv[s][k].y; xv[k].z += yv[s][k].z; xv[k].w += yv[s][k].w;
      }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (own[k]) *reinterpret_cast<float4*>(x + 4 * (t + T * k)) = xv[k];
  }
  if constexpr (NY < 0) {
    for (int s = 0; s < -NY; ++s) {
      const float* src = (ys.p[0] ? ys.p[s] : Y + s * y_stride) + (size_t)row * d;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!own[k]) continue;
        const float4 y = __ldcs(reinterpret_cast<const float4*>(src + 4 * (t + T * k)));
        xv[k].x += y.x; xv[k].y += y.y; xv[k].z += y.z; xv[k].w += y.w;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (own[k]) *reinterpret_cast<float4*>(x + 4 * (t + T * k)) = xv[k];
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) ss += xv[k].x * xv[k].x + xv[k].y * xv[k].y + xv[k].z * xv[k].z + xv[k].w * xv[k].w;
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o, 32);
  const int nw = (blockDim.x + 31) >> 5;
  if (nw > 1) {
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < nw ? red[threadIdx.x] : 0.f;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
      if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    ss = red[0];
  }
  const float inv = rsqrtf(ss / (float)d + eps);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (!own[k]) continue;
    const int e = 4 * (t + T * k);
    const uint2 gu = *reinterpret_cast<const uint2*>(g + e);
    const float xs[4] = {xv[k].x, xv[k].y, xv[k].z, xv[k].w};
    const uint32_t gw[2] = {gu.x, gu.y};
    uint32_t o[2], r[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float y0 = xs[2 * q] * inv * __uint_as_float(gw[q] << 16);
      const float y1 = xs[2 * q + 1] * inv * __uint_as_float(gw[q] & 0xFFFF0000u);
      __nv_bfloat162 p = __floats2bfloat162_rn(y0, y1);
      o[q] = *reinterpret_cast<uint32_t*>(&p);
      const float h0 = __uint_as_float(o[q] << 16), h1 = __uint_as_float(o[q] & 0xFFFF0000u);
      __nv_bfloat162 pq = __floats2bfloat162_rn(y0 - h0, y1 - h1);
      r[q] = *reinterpret_cast<uint32_t*>(&pq);
    }
    if (split) {
      *reinterpret_cast<uint2*>(out + (size_t)(2 * row) * d + e) = make_uint2(o[0], o[1]);
      *reinterpret_cast<uint2*>(out + (size_t)(2 * row + 1) * d + e) = make_uint2(r[0], r[1]);
    } else if (ys.nout) {
      // NEXT-F4 all-gather: this rank's normalised row into every rank's copy (NVLink stores)
      for (int p = 0; p < ys.nout; ++p) *reinterpret_cast<uint2*>(ys.outp[p] + (size_t)row * d + e) = make_uint2(o[0], o[1]);
    } else {
      *reinterpret_cast<uint2*>(out + (size_t)row * d + e) = make_uint2(o[0], o[1]);
    }
  }
}

// ------------------------------------------------------------------------- K4b QKV RoPE/scatter
// One thread per 4 consecutive rotate-half pairs (i..i+3, i+hd/2..i+hd/2+3) of one q or k head at
// position row_pos (amb. A14), or per 4 consecutive v elements; float4 loads of every K-split
// partial (summed in split order), fp16 stores.
__global__ void k_qkv_rope(const __grid_constant__ RopeArgs r) {
  pdl_begin();
  const int row = blockIdx.y;
  const int hd = r.hd, half = hd >> 1, hq = half >> 2;    // 4-pair groups per head
  const int qkv = (r.H + 2 * r.KV) * hd;
  const int ngroups = (r.H + r.KV) * hq;
  const int nv4 = r.KV * hd / 4;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ngroups + nv4) return;
  const float* y = r.Y + (size_t)row * qkv;
  auto ld4 = [&](int f) {
    float4 v = __ldcs(reinterpret_cast<const float4*>(y + f));
    for (int s = 1; s < r.nY; ++s) {
      const float4 w = __ldcs(reinterpret_cast<const float4*>(y + s * r.y_stride + f));
      v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
    }
    return v;
  };
  auto st4 = [](f16* dst, float a, float b, float c, float d) {
    __half2 p0 = __floats2half2_rn(a, b), p1 = __floats2half2_rn(c, d);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&p0);
    u.y = *reinterpret_cast<uint32_t*>(&p1);
    *reinterpret_cast<uint2*>(dst) = u;
  };
  if (e < ngroups) {
    const int head = e / hq, i = (e % hq) * 4;
    const int f1 = head * hd + i;
    const float4 x1 = ld4(f1), x2 = ld4(f1 + half);
    const int pos = r.row_pos[row];
    const float4 c = *reinterpret_cast<const float4*>(r.rope_cos + (size_t)pos * half + i);
    const float4 sn = *reinterpret_cast<const float4*>(r.rope_sin + (size_t)pos * half + i);
    f16* dst;
    if (head < r.H) {
      dst = r.Q + (size_t)row * r.H * hd + head * hd;
    } else {
      dst = r.tree_kv + ((((size_t)r.layer * 2 + 0) * r.KV + (head - r.H)) * r.R_cap + row) * hd;
    }
    st4(dst + i, x1.x * c.x - x2.x * sn.x, x1.y * c.y - x2.y * sn.y, x1.z * c.z - x2.z * sn.z, x1.w * c.w - x2.w * sn.w);
    st4(dst + i + half, x2.x * c.x + x1.x * sn.x, x2.y * c.y + x1.y * sn.y, x2.z * c.z + x1.z * sn.z,
        x2.w * c.w + x1.w * sn.w);
  } else {
    const int ve = (e - ngroups) * 4;
    const int kvh = ve / hd, dd = ve % hd;
    const float4 x = ld4((r.H + r.KV) * hd + ve);
    st4(r.tree_kv + ((((size_t)r.layer * 2 + 1) * r.KV + kvh) * r.R_cap + row) * hd + dd, x.x, x.y, x.z, x.w);
  }
}

// ----------------------------------------------------------------------- K9b argmax reduction
// One warp per row over the per-128-vocab-tile partials.  Order (value desc, index asc).
__global__ void k_lm_reduce(const float* __restrict__ pv, const int* __restrict__ pi, int R, int ntiles,
                            int* __restrict__ y, float* __restrict__ score, int* __restrict__ row_target,
                            float* __restrict__ row_score) {
  pdl_begin();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= R) return;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = lane; t < ntiles; t += 32) {
    const float v = pv[(size_t)row * ntiles + t];
    const int i = pi[(size_t)row * ntiles + t];
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float v = __shfl_xor_sync(0xffffffff, best, o);
    const int i = __shfl_xor_sync(0xffffffff, bi, o);
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
  if (lane == 0) {
    y[row] = bi;
    score[row] = best;
    if (row_target) row_target[row] = bi;
    if (row_score) row_score[row] = best;
  }
}

// ------------------------------------------------------------- K9c hi-only LM head refinement
// One 4-warp block per row (RefineArgs in internal.h).  The window uses the row's own ||hi||_2,
// ||lo||_2 (read here, so tensor-parallel ranks need no extra collective) and the shard's
// max_v ||W_v||_2.  The warps split the tiles (max, candidate gathering into a shared list) and the
// row (norms), then rescore the list kRefineBatch LM-head rows at a time, warp w taking batches
// w, w+4, ...; the per-warp winners are combined in (score desc, id asc) order, so the result does
// not depend on the gathering order.
constexpr int kRefineBatch = 4;
constexpr int kRefineWarps = 4;
constexpr int kRefineList = 1024;

__global__ void __launch_bounds__(kRefineWarps * 32) k_lm_refine(const __grid_constant__ RefineArgs a) {
  pdl_begin();
  __shared__ int s_list[kRefineList];
  __shared__ int s_n, s_over;
  __shared__ float s_red[3][kRefineWarps];
  __shared__ float s_best[kRefineWarps];
  __shared__ int s_bi[kRefineWarps];
  const int row = blockIdx.x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const size_t base = (size_t)row * a.ntiles;
  const float* pv = a.part_val + base;
  const float* pv2 = a.part_val2 + base;
  const float* pv3 = a.part_val3 + base;
  const uint4* hi = reinterpret_cast<const uint4*>(a.hf + (size_t)(2 * row) * a.d);
  const uint4* lo = reinterpret_cast<const uint4*>(a.hf + (size_t)(2 * row + 1) * a.d);
  const int nv = a.d / 8;
  if (tid == 0) { s_n = 0; s_over = 0; }
  // ---- phase 1: best hi score of the row, ||hi||, ||lo|| (all loads of a batch before any use)
  float M = -INFINITY, sh = 0.f, sl = 0.f;
  for (int t0 = 0; t0 < a.ntiles; t0 += 128 * 4) {
    float v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int t = t0 + tid + 128 * i;
      v[i] = t < a.ntiles ? __ldg(pv + t) : -INFINITY;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) M = fmaxf(M, v[i]);
  }
  for (int e0 = 0; e0 < nv; e0 += 128 * 2) {
    uint4 h[2], l[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = e0 + tid + 128 * i;
      h[i] = e < nv ? __ldg(hi + e) : make_uint4(0u, 0u, 0u, 0u);
      l[i] = e < nv ? __ldg(lo + e) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint32_t hw[4] = {h[i].x, h[i].y, h[i].z, h[i].w}, lw[4] = {l[i].x, l[i].y, l[i].z, l[i].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float h0 = __uint_as_float(hw[k] << 16), h1 = __uint_as_float(hw[k] & 0xFFFF0000u);
        const float l0 = __uint_as_float(lw[k] << 16), l1 = __uint_as_float(lw[k] & 0xFFFF0000u);
        sh = fmaf(h0, h0, fmaf(h1, h1, sh));
        sl = fmaf(l0, l0, fmaf(l1, l1, sl));
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    sh += __shfl_xor_sync(0xffffffffu, sh, o);
    sl += __shfl_xor_sync(0xffffffffu, sl, o);
  }
  if (lane == 0) { s_red[0][w] = M; s_red[1][w] = sh; s_red[2][w] = sl; }
  __syncthreads();
  M = -INFINITY; sh = 0.f; sl = 0.f;
#pragma unroll
  for (int i = 0; i < kRefineWarps; ++i) { M = fmaxf(M, s_red[0][i]); sh += s_red[1][i]; sl += s_red[2][i]; }
  // |score_hi(v) - score(v)| <= (||lo|| + rho) wmax scale, rho = d 2^-24 (||hi|| + ||lo||) bounds
  // the fp32 accumulation error of either evaluation; + a few ulps of |M| for the final rounding
  const float nh = sqrtf(sh) * 1.0001f, nl = sqrtf(sl) * 1.0001f;
  const float scale = a.sample ? a.inv_t : 1.f;
  const float rho = (float)a.d * 5.9604645e-08f * (nh + nl);
  const float win = 2.f * (nl + rho) * a.wmax * scale + 8.f * 1.1920929e-07f * fabsf(M) + 1e-6f;
  const float thr = M - win;
  // ---- phase 2: gather the candidates (a tile's best / second, or all of a tile whose third
  // score is inside the window)
  auto push = [&](int v) {
    const int at = atomicAdd(&s_n, 1);
    if (at < kRefineList) s_list[at] = v;
    else s_over = 1;
  };
  for (int t = tid; t < a.ntiles; t += kRefineWarps * 32) {
    if (__ldg(pv + t) < thr) continue;
    if (__ldg(pv3 + t) >= thr) {
      const int v1 = min(a.vocab, (t + 1) * 128);
      for (int v = t * 128; v < v1; ++v) push(v);
    } else {
      push(__ldg(a.part_idx + base + t) - a.vocab_off);
      if (__ldg(pv2 + t) >= thr) push(__ldg(a.part_idx2 + base + t) - a.vocab_off);
    }
  }
  __syncthreads();
  const int n = min(s_n, kRefineList);
  const bool over = s_over != 0;
  // ---- phase 3: exact (hi + lo) . W_v (+ Gumbel) of the candidates, kRefineBatch rows of W per pass
  const int req = a.row_req[row];
  const uint64_t ses = a.req_session[req];
  const uint32_t k0 = a.seed_lo ^ a.req_round[req], slot = (uint32_t)a.row_slot[row];
  float best = -INFINITY;
  int bi = 0x7fffffff;
  auto rescore = [&](auto id_of, int cnt, int c_begin, int c_step) {
    for (int c0 = c_begin * kRefineBatch; c0 < cnt; c0 += c_step * kRefineBatch) {
      const uint4* wr[kRefineBatch];
      float acc[kRefineBatch];
#pragma unroll
      for (int bb = 0; bb < kRefineBatch; ++bb) {
        wr[bb] = reinterpret_cast<const uint4*>(a.w + (size_t)id_of(min(c0 + bb, cnt - 1)) * a.d);
        acc[bb] = 0.f;
      }
      for (int e0 = 0; e0 < nv; e0 += 64) {
        uint4 hh[2], ll[2], ww[2][kRefineBatch];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int e = e0 + lane + 32 * i;
          const bool ok = e < nv;
          hh[i] = ok ? __ldg(hi + e) : make_uint4(0u, 0u, 0u, 0u);
          ll[i] = ok ? __ldg(lo + e) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int bb = 0; bb < kRefineBatch; ++bb) ww[i][bb] = ok ? __ldg(wr[bb] + e) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const uint32_t hw[4] = {hh[i].x, hh[i].y, hh[i].z, hh[i].w}, lw[4] = {ll[i].x, ll[i].y, ll[i].z, ll[i].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            // hi + lo is exact in fp32 (bf16 + bf16 below half an ulp of hi)
            const float y0 = __uint_as_float(hw[k] << 16) + __uint_as_float(lw[k] << 16);
            const float y1 = __uint_as_float(hw[k] & 0xFFFF0000u) + __uint_as_float(lw[k] & 0xFFFF0000u);
#pragma unroll
            for (int bb = 0; bb < kRefineBatch; ++bb) {
              const uint32_t wv = k == 0 ? ww[i][bb].x : (k == 1 ? ww[i][bb].y : (k == 2 ? ww[i][bb].z : ww[i][bb].w));
              acc[bb] = fmaf(y0, __uint_as_float(wv << 16), acc[bb]);
              acc[bb] = fmaf(y1, __uint_as_float(wv & 0xFFFF0000u), acc[bb]);
            }
          }
        }
      }
#pragma unroll
      for (int bb = 0; bb < kRefineBatch; ++bb) {
        float v = acc[bb];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (c0 + bb >= cnt) continue;
        const int vg = a.vocab_off + id_of(c0 + bb);
        if (a.sample) {
          const U4 r = philox4x32_10(U4{(uint32_t)vg >> 2, slot, (uint32_t)ses, (uint32_t)(ses >> 32)}, k0, a.seed_hi);
          v = v * a.inv_t + gumbel_of_word(u4_word(r, vg & 3));
        }
        if (v > best || (v == best && vg < bi)) { best = v; bi = vg; }
      }
    }
  };
  rescore([&](int c) { return s_list[c]; }, n, w, kRefineWarps);
  if (over && w == 0) {
    // more than kRefineList candidates (only when whole tiles pile up): warp 0 rescores every id of
    // every tile inside the window; duplicates of the list are harmless (same score, same id)
    for (int t = 0; t < a.ntiles; ++t) {
      if (__ldg(pv + t) < thr) continue;
      const int v0 = t * 128, cnt = min(a.vocab, v0 + 128) - v0;
      rescore([&](int c) { return v0 + c; }, cnt, 0, 1);
    }
  }
  if (lane == 0) { s_best[w] = best; s_bi[w] = bi; }
  __syncthreads();
  if (tid == 0) {
    for (int i = 1; i < kRefineWarps; ++i)
      if (s_best[i] > best || (s_best[i] == best && s_bi[i] < bi)) { best = s_best[i]; bi = s_bi[i]; }
    a.y[row] = bi;
    a.score[row] = best;
    if (a.row_target) a.row_target[row] = bi;
    if (a.row_score) a.row_score[row] = best;
  }
}

__global__ void k_row_norm_max(const bf16* __restrict__ w, int rows, int d, float* __restrict__ out) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint4* wr = reinterpret_cast<const uint4*>(w + (size_t)row * d);
  float s = 0.f;
  for (int e = lane; e < d / 8; e += 32) {
    const uint4 x = wr[e];
    const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float a0 = __uint_as_float(xw[k] << 16), a1 = __uint_as_float(xw[k] & 0xFFFF0000u);
      s = fmaf(a0, a0, fmaf(a1, a1, s));
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  // non-negative floats order like their bit patterns
  if (lane == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(sqrtf(s)));
}

// ------------------------------------------------------------------------------ K10 walk
// One warp per request; lane l examines nodes l and l+32 (N <= 64 for valid requests).
__global__ void k_walk(const __grid_constant__ WalkArgs w) {
  pdl_begin();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= w.B) return;
  const int n0 = w.node_offset[r];
  const int N = w.node_offset[r + 1] - n0;
  const int row0 = n0 + r;
  if (w.status[r] != SPECEDGE_REQ_OK) {
    if (lane == 0) {
      w.accepted_len[r] = 0;
      w.bonus[r] = -1;
    }
    return;
  }
  if (w.force_chain) {   // prefill: accept the whole chain
    for (int i = lane; i < N; i += 32) {
      w.accepted_token[n0 + i] = w.token[n0 + i];
      w.accepted_node[n0 + i] = i;
    }
    if (lane == 0) {
      w.accepted_len[r] = N;
      w.bonus[r] = -1;
    }
    return;
  }
  int par[2], tok[2];
  for (int k = 0; k < 2; ++k) {
    const int i = lane + 32 * k;
    par[k] = i < N ? w.parent[n0 + i] : -2;
    tok[k] = i < N ? w.token[n0 + i] : -1;
  }
  int cur = -1, a = 0;
  while (true) {
    const int want = w.y[row0 + cur + 1];
    int found = -1;
    for (int k = 0; k < 2; ++k) {
      const unsigned m = __ballot_sync(0xffffffff, par[k] == cur && tok[k] == want);
      if (m && found < 0) found = (__ffs(m) - 1) + 32 * k;
    }
    if (found < 0) break;
    if (lane == 0) {
      w.accepted_token[n0 + a] = want;
      w.accepted_node[n0 + a] = found;
    }
    ++a;
    cur = found;
  }
  if (lane == 0) {
    w.accepted_len[r] = a;
    w.bonus[r] = w.y[row0 + cur + 1];
  }
}

// ----------------------------------------------------------------------------- K11 commit
// grid (B, layers).  Copies K/V of slot 0 and of the accepted slots (in path order) from the tree
// scratch to cache positions L, L+1, ..., L+a.  Scratch and pages are distinct buffers, so the
// copy has no aliasing hazard.  Only if the cached length is still the one
// this verify saw (idempotence guard).
__global__ void k_commit(const __grid_constant__ CommitArgs c) {
  pdl_begin();
  const int r = blockIdx.x, layer = blockIdx.y;
  if (c.status[r] != SPECEDGE_REQ_OK) return;
  const int h = c.req_h[r];
  const int L = c.req_L[r];
  if (c.cache_len[h] != L) return;
  const int a = c.accepted_len[r];
  const int n0 = c.node_offset[r];
  const int row0 = c.req_row0[r];
  const int vec_per_row = c.hd / 8;           // uint4 per head row
  const int per_tok = 2 * c.KV * vec_per_row;
  for (int idx = threadIdx.x; idx < (a + 1) * per_tok; idx += blockDim.x) {
    const int j = idx / per_tok;
    const int rem = idx % per_tok;
    const int kvsel = rem / (c.KV * vec_per_row);
    const int g = (rem / vec_per_row) % c.KV;
    const int v = rem % vec_per_row;
    const int slot = j == 0 ? 0 : c.accepted_node[n0 + j - 1] + 1;
    const size_t src = ((((size_t)layer * 2 + kvsel) * c.KV + g) * c.R_cap + row0 + slot) * c.hd;
    const int pos = L + j;
    const int page = c.block_table[(size_t)h * c.max_pages_per_seq + pos / kPage];
    const size_t dst = (((((size_t)layer * c.num_pages + page) * 2 + kvsel) * c.KV + g) * kPage + pos % kPage) * c.hd;
    reinterpret_cast<uint4*>(c.pool + dst)[v] = reinterpret_cast<const uint4*>(c.tree_kv + src)[v];
  }
}

__global__ void k_commit_finalize(const __grid_constant__ CommitArgs c) {
  pdl_begin();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= c.B || c.status[r] != SPECEDGE_REQ_OK) return;
  const int h = c.req_h[r];
  if (c.cache_len[h] != c.req_L[r]) {
    c.status[r] = SPECEDGE_REQ_E_CONTEXT;   // already committed
    return;
  }
  c.cache_len[h] = c.req_L[r] + c.accepted_len[r] + 1;
}

// cache_len[handle[i]] = len[i] for a batch of up to kSetLenBatch sessions passed by value (one
// tiny launch, capturable in a CUDA graph; no host staging)
__global__ void k_set_len(int* __restrict__ cache_len, const __grid_constant__ SetLenArgs a) {
  pdl_begin();
  const int i = threadIdx.x;
  if (i < a.n) cache_len[a.handle[i]] = a.len[i];
}

// ------------------------------------------------------- NEXT-F2 dense-q speculative sampling
// One warp per row: lse = M + log sum_t s_t exp(m_t - M) over the PQ1 tile partials; q row of the
// slot = the node drawn there (slot s < N: node s of a chain), -1 for the last slot.
__global__ void k_pq_lse(const __grid_constant__ PqArgs a) {
  pdl_begin();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= a.R) return;
  float m = -INFINITY;
  for (int t = lane; t < a.ntiles; t += 32) m = fmaxf(m, a.part_m[(size_t)row * a.ntiles + t]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
  float sm = 0.f;
  if (m > -INFINITY)
    for (int t = lane; t < a.ntiles; t += 32)
      sm += a.part_s[(size_t)row * a.ntiles + t] * __expf(a.part_m[(size_t)row * a.ntiles + t] - m);
  for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffff, sm, o);
  if (lane == 0) {
    a.lse[row] = m + __logf(sm);
    const int r = a.row_req[row], sl = a.row_slot[row];
    const int n0 = a.node_offset[r], N = a.node_offset[r + 1] - n0;
    a.row_qnode[row] = sl < N ? n0 + sl : -1;
  }
}

// Leviathan et al. over a sampled chain (oracle/pq.py): node i (drawn from q_i) is accepted iff
// u(slot i) < p_i(x) / q_i(x); the first rejection's bonus is the residual draw of that slot,
// the bonus after full acceptance the Gumbel-max of p at the last slot.  u(slot): Philox word 0 of
// counter (slot, 'ACPT', lo32(session), hi32(session)), key (lo32(seed) ^ round, hi32(seed)).
__global__ void k_pq_walk(const __grid_constant__ PqArgs a) {
  pdl_begin();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.B) return;
  const int n0 = a.node_offset[r];
  const int N = a.node_offset[r + 1] - n0;
  const int row0 = n0 + r;
  bool ok = a.status[r] == SPECEDGE_REQ_OK;
  if (ok)
    for (int i = 0; i < N; ++i)
      if (a.parent[n0 + i] != i - 1) {   // dense-q mode verifies chains only
        a.status[r] = SPECEDGE_REQ_E_UNSUPPORTED;
        ok = false;
        break;
      }
  if (!ok) {
    a.accepted_len[r] = 0;
    a.bonus[r] = -1;
    return;
  }
  const uint64_t ses = a.req_session[r];
  const uint32_t k0 = a.seed_lo ^ a.req_round[r];
  int acc = 0, bonus = -1;
  for (int i = 0; i < N; ++i) {
    const int x = a.token[n0 + i];
    const float qx = a.draft_q[(size_t)(n0 + i) * a.V + x];
    const float ratio = qx > 0.f ? a.pchild[row0 + i] / qx : INFINITY;
    const U4 w = philox4x32_10(U4{(uint32_t)i, 0x41435054u, (uint32_t)ses, (uint32_t)(ses >> 32)}, k0, a.seed_hi);
    const float u = (float)((w.x >> 8) | 1u) * 5.9604644775390625e-08f;   // exact, in (0, 1)
    if (u < ratio) {
      a.accepted_token[n0 + acc] = x;
      a.accepted_node[n0 + acc] = i;
      ++acc;
    } else {
      bonus = a.resid_y[row0 + i];
      break;
    }
  }
  if (acc == N) bonus = a.y[row0 + N];
  a.accepted_len[r] = acc;
  a.bonus[r] = bonus;
}

// ------------------------------------------------------------------------ K12 weight init
// Element (lrow, col) of a logical weight = bf16(f32(i24 * scale)) with i24 from Philox counter
// (idx >> 2, tensor_id, layer, 'WEIG'), idx = lrow * cols + col, word idx & 3 (oracle/model.py O1).
__global__ void k_init_weights(const __grid_constant__ InitArgs a) {
  const long long total4 = a.rows * a.cols / 4;
  for (long long g4 = blockIdx.x * (long long)blockDim.x + threadIdx.x; g4 < total4;
       g4 += (long long)gridDim.x * blockDim.x) {
    const long long prow = g4 * 4 / a.cols;
    const long long col = g4 * 4 % a.cols;
    int tid = a.tid0;
    long long lrow = prow + a.off0;
    float scale = a.scale0;
    if (a.layout == INIT_QKV) {
      if (prow < a.rows0) { tid = a.tid0; lrow = a.off0 + prow; scale = a.scale0; }
      else if (prow < a.rows0 + a.rows1) { tid = a.tid1; lrow = a.off1 + prow - a.rows0; scale = a.scale1; }
      else { tid = a.tid2; lrow = a.off2 + prow - a.rows0 - a.rows1; scale = a.scale2; }
    } else if (a.layout == INIT_GATEUP) {
      const long long blk = prow / 128, within = prow % 128;
      if (within < 64) { tid = a.tid0; lrow = a.off0 + blk * 64 + within; scale = a.scale0; }
      else { tid = a.tid1; lrow = a.off0 + blk * 64 + within - 64; scale = a.scale1; }
    }
    // global element index (multiple of 4: col0, gcols and cols are multiples of 4)
    const unsigned long long idx = (unsigned long long)lrow * a.gcols + a.col0 + col;
    const U4 r = philox4x32_10(U4{(uint32_t)(idx >> 2), (uint32_t)tid, (uint32_t)a.layer, 0x57454947u}, a.k0, a.k1);
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    uint16_t out[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float v;
      if (a.gain) v = __fadd_rn(__fmul_rn(philox_i24(w[k]), 2.98023223876953125e-08f), 1.0f);
      else v = __fmul_rn(philox_i24(w[k]), scale);
      out[k] = f32_to_bf16_bits(v);
    }
    uint2 pk;
    pk.x = (uint32_t)out[0] | ((uint32_t)out[1] << 16);
    pk.y = (uint32_t)out[2] | ((uint32_t)out[3] << 16);
    *reinterpret_cast<uint2*>(a.dst + prow * a.cols + col) = pk;
  }
}

// ---------------------------------------------------------------------- K13 synthetic KV
// element e = head*hd + j of token t: Philox counter (e>>2, t, layer*2 + kv, stream ^ 'KVFI').
__global__ void k_kv_fill(f16* pool, const int* __restrict__ block_row, int layers, int num_pages, int KV,
                          int hd, int n_tokens, uint32_t k0, uint32_t k1, uint32_t stream_id, int kv_head0) {
  // kv_head0: global index of local kv head 0 (tensor-parallel pool shard); the Philox counter
  // uses the global element index, so a shard holds exactly the global cache's values
  const int per_tok4 = KV * hd / 4;
  const int e4_off = kv_head0 * hd / 4;
  const long long total = (long long)n_tokens * layers * 2 * per_tok4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int e4 = (int)(i % per_tok4);
    long long rest = i / per_tok4;
    const int kvsel = (int)(rest % 2);
    rest /= 2;
    const int layer = (int)(rest % layers);
    const int t = (int)(rest / layers);
    const U4 r = philox4x32_10(U4{(uint32_t)(e4 + e4_off), (uint32_t)t, (uint32_t)((layer << 1) | kvsel), stream_id ^ 0x4B564649u}, k0, k1);
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    uint16_t out[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = __half_as_ushort(__float2half_rn(__fmul_rn(philox_i24(w[k]), 1.1920928955078125e-07f)));
    const int e = e4 * 4;
    const int g = e / hd, j = e % hd;
    const int page = block_row[t / kPage];
    const size_t dst = (((((size_t)layer * num_pages + page) * 2 + kvsel) * KV + g) * kPage + t % kPage) * hd + j;
    uint2 pk;
    pk.x = (uint32_t)out[0] | ((uint32_t)out[1] << 16);
    pk.y = (uint32_t)out[2] | ((uint32_t)out[3] << 16);
    *reinterpret_cast<uint2*>(pool + dst) = pk;
  }
}

}  // namespace

cudaError_t prep_launch(const PrepArgs& p, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  CK_RET(launch_k(k_prep, dim3(p.B), dim3(64), 0, st, p));
  return cudaGetLastError();
}
cudaError_t embed_launch(const bf16* E, const int* row_tok, float* X, int R, int d, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  CK_RET(launch_k(k_embed, dim3(R), dim3(128), 0, st, E, row_tok, X, d));
  return cudaGetLastError();
}
cudaError_t rmsnorm_launch(float* X, const float* Y, int nY, size_t y_stride, const bf16* g, bf16* out, int R, int d,
                           float eps, cudaStream_t st, int* launches, int split, const RmsSrc* ys) {
  if (launches) ++*launches;
  const int threads = (d / 16 + 31) & ~31;   // whole warps; d % 64 == 0 and d <= 16384 (model creation)
  const RmsSrc src = ys ? *ys : RmsSrc{};
  if (carveout_mode() == 2) {
    static PerDeviceOnce once;
    if (once.first()) {
      carveout_skip(reinterpret_cast<const void*>(k_rmsnorm<0>));
      carveout_skip(reinterpret_cast<const void*>(k_rmsnorm<1>));
      carveout_skip(reinterpret_cast<const void*>(k_rmsnorm<2>));
      carveout_skip(reinterpret_cast<const void*>(k_rmsnorm<3>));
      carveout_skip(reinterpret_cast<const void*>(k_rmsnorm<4>));
    }
  }
  switch (nY) {
    case 0: CK_RET(launch_k(k_rmsnorm<0>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    case 1: CK_RET(launch_k(k_rmsnorm<1>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    case 2: CK_RET(launch_k(k_rmsnorm<2>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    case 3: CK_RET(launch_k(k_rmsnorm<3>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    case 4: CK_RET(launch_k(k_rmsnorm<4>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    case 5: CK_RET(launch_k(k_rmsnorm<-5>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    case 6: CK_RET(launch_k(k_rmsnorm<-6>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    case 7: CK_RET(launch_k(k_rmsnorm<-7>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    case 8: CK_RET(launch_k(k_rmsnorm<-8>, dim3(R), dim3(threads), 0, st, X, Y, y_stride, g, out, d, eps, split, src)); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
cudaError_t qkv_rope_launch(const RopeArgs& r, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  const int items = (r.H + r.KV) * (r.hd / 8) + r.KV * r.hd / 4;   // head_dim >= 16
  CK_RET(launch_k(k_qkv_rope, dim3((items + 127) / 128, r.R), dim3(128), 0, st, r));
  return cudaGetLastError();
}
cudaError_t lm_reduce_launch(const float* pv, const int* pi, int R, int ntiles, int* y, float* score,
                             int* row_target, float* row_score, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  CK_RET(launch_k(k_lm_reduce, dim3((R + 3) / 4), dim3(128), 0, st, pv, pi, R, ntiles, y, score, row_target, row_score));
  return cudaGetLastError();
}
cudaError_t lm_refine_launch(const RefineArgs& a, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  CK_RET(launch_k(k_lm_refine, dim3(a.R), dim3(kRefineWarps * 32), 0, st, a));
  return cudaGetLastError();
}
cudaError_t row_norm_max_launch(const bf16* w, int rows, int d, float* out, cudaStream_t st) {
  CK_RET(cudaMemsetAsync(out, 0, sizeof(float), st));
  k_row_norm_max<<<(rows + 7) / 8, 256, 0, st>>>(w, rows, d, out);
  return cudaGetLastError();
}
cudaError_t walk_launch(const WalkArgs& w, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  CK_RET(launch_k(k_walk, dim3((w.B + 3) / 4), dim3(128), 0, st, w));
  return cudaGetLastError();
}
cudaError_t commit_launch(const CommitArgs& c, cudaStream_t st, int* launches) {
  if (launches) *launches += 2;
  CK_RET(launch_k(k_commit, dim3(c.B, c.layers), dim3(256), 0, st, c));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CK_RET(launch_k(k_commit_finalize, dim3((c.B + 127) / 128), dim3(128), 0, st, c));
  return cudaGetLastError();
}
cudaError_t pq_lse_launch(const PqArgs& a, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  CK_RET(launch_k(k_pq_lse, dim3((a.R + 3) / 4), dim3(128), 0, st, a));
  return cudaGetLastError();
}
cudaError_t pq_walk_launch(const PqArgs& a, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  CK_RET(launch_k(k_pq_walk, dim3((a.B + 127) / 128), dim3(128), 0, st, a));
  return cudaGetLastError();
}
cudaError_t set_len_launch(int* cache_len, const SetLenArgs& a, cudaStream_t st) {
  CK_RET(launch_k(k_set_len, dim3(1), dim3(kSetLenBatch), 0, st, cache_len, a));
  return cudaGetLastError();
}
cudaError_t init_weights_launch(const InitArgs& a, cudaStream_t st) {
  const long long total4 = a.rows * a.cols / 4;
  const int blocks = (int)std::min<long long>((total4 + 255) / 256, 148 * 16);
  k_init_weights<<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t kv_fill_launch(f16* pool, const int* block_row, int layers, int num_pages, int KV, int hd, int n_tokens,
                           uint32_t k0, uint32_t k1, uint32_t stream_id, int kv_head0, cudaStream_t st) {
  const long long total = (long long)n_tokens * layers * 2 * (KV * hd / 4);
  if (total == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  k_kv_fill<<<blocks, 256, 0, st>>>(pool, block_row, layers, num_pages, KV, hd, n_tokens, k0, k1, stream_id, kv_head0);
  return cudaGetLastError();
}

}  // namespace se
