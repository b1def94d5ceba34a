// Tree-masked paged split-KV attention on tcgen05 ("custom attention
// masking for each token sequence in the batch ... without cross-sequence interference").
//
// Work item = (request r, kv head g, a range of the request's 64-key sub-tiles: pages of the paged
// cache, then the tree slots from the tree K/V scratch, masked by the uint64 ancestor-or-self
// bitmask).  Query rows of an item are the request's S slots x the G query heads sharing kv head g
// (row = s*G + j), cut into 128-row M-tiles of G*floor(128/G) rows.  Sub-tiles stream through a
// TMA ring (hd 128: 5 stages with two Q tiles, 6 with one).
//   static mode:   one CTA per (r, g, chunk of pages_per_split pages; the tree in the last chunk)
//   balanced mode: a persistent grid; the concatenated (r, g) sub-tile sequences are split
//                  evenly over the CTAs, the pipeline runs on across a CTA's items, and for groups
//                  of <= 128 rows the last CTA to finish a chunk of (r, g) merges all its chunks
//                  (long contexts: cfg5), otherwise k_attn_combine does.
//
// Two "units" share the CTA; a unit = one softmax warpgroup + its TMEM (two 64-column S buffers
// + a 128-column O accumulator).  A pass streams the KV once:
//   pair pass   (>= 2 M-tiles left): unit u owns M-tile 2p+u and consumes every sub-tile, so two
//               M-tiles share one KV read (cfg2's 132 rows = 1 pass instead of 2);
//   single pass (last M-tile alone): both units work on the same M-tile, unit u taking sub-tiles
//               j = u mod 2 with its own running max / sum / O (an in-CTA 2-way KV split), merged
//               in the epilogue.
// Within a unit, S is double-buffered at sub-tile granularity: while the warps turn S(k) into P(k),
// the tensor core computes S(k+1); S(k+2) overwrites P(k) right after PV(k) (in-order tcgen05).
//
//   warp 0      TMA producer: Q tiles (3-D map over Q[R][H][hd]), K/V sub-tiles (2-D maps)
//   warp 1      TMEM allocator + MMA issuer of unit 0; warp 10: MMA issuer of unit 1 (one elected
//               thread each, so one unit's barrier waits never delay the other's issue):
//                 S_u  = Q_u K^T      kind::f16, M=128 N=64, A,B from smem (K-major, SW128)
//                 O_u += P_u V        A = P (fp16) from TMEM, B = V from smem (MN-major, SW128)
//   warps 2-5   unit 0 softmax + epilogue (one thread = one query row: no cross-thread reduction)
//   warps 6-9   unit 1 softmax + epilogue
//
// Softmax in the log2 domain with a lazily updated running max (O is rescaled only when the max
// grows by more than 8, exact because l uses the same max).  P enters PV as fp16 (11-bit
// significand: ~2e-4 relative error; bf16 P would give ~1.5e-3, SURVEY amb. A12); q, k, v are fp16
// (DESIGN.md R-precision).
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

namespace se {

namespace {

constexpr int kWarps = 11;      // producer, MMA (unit 0), 2 units x 4 softmax/epilogue warps, MMA (unit 1)
constexpr int kThreads = kWarps * 32;
// K/V ring depth (64-key sub-tiles): whatever the 227 KB of shared memory leaves after NQ Q tiles
// and ~3 KB of barriers / masks / merge scalars (hd 128: 5 stages with two Q tiles, 6 with one;
// hd 64: 12).  The ring is the only source of memory-level parallelism: at steady state the two
// units hold about four sub-tiles, the rest are in flight.
constexpr int kSmemMax = 227 * 1024;
constexpr int kSmemAux = 3 * 1024;
__host__ __device__ constexpr int ring_stages(int hd, int nq) {
  return (kSmemMax - kSmemAux - nq * 128 * hd * 2) / (2 * 64 * hd * 2) > 12
             ? 12
             : (kSmemMax - kSmemAux - nq * 128 * hd * 2) / (2 * 64 * hd * 2);
}
#ifndef SPECEDGE_EMU8
#define SPECEDGE_EMU8 0
#endif
constexpr int kEmu8 = SPECEDGE_EMU8;   // exponentials per 8 on exp2_fma (rest ex2.approx); measured no gain at 2-4 (profiles/README.md)
constexpr int kPrefetchDefault = 0;   // L2 prefetch distance (sub-tiles) ahead of the ring; env SPECEDGE_ATTN_PREFETCH

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
__device__ __forceinline__ void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
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

// 2^x on the FMA/ALU pipes (for x <= 8): round-to-nearest split x = n + f via the 1.5*2^23 trick,
// degree-3 fit of 2^f on [-1/2, 1/2] (max relative error 1.1e-4, below the fp16 rounding of P),
// exponent add for 2^n.  Used for a fraction of the softmax exponentials so that the MUFU pipe
// (16 ex2/clk/SM on B200) is not the bound (the FA4 idea).
__device__ __forceinline__ float exp2_fma(float x) {
  x = fmaxf(x, -127.0f);
  const float t = x + 12582912.0f;
  const float nf = t - 12582912.0f;
  const float f = x - nf;
  float p = fmaf(f, 0.054592829f, 0.24221838f);
  p = fmaf(p, f, 0.69336867f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ void tma_prefetch_l2_2d(const CUtensorMap* m, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1)
               : "memory");
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
  bf16* O;          // final normalised output of single-chunk items (bf16), or nullptr
  float* O_f32;     // optional fp32 normalised output (debug)
  int slots_per_mt; // floor(128 / G)
  int prefetch;     // L2 prefetch distance in sub-tiles (0: off)
  unsigned long long* trace;   // debug (env SPECEDGE_ATTN_TRACE): clock64 stamps of CTA 0, else null
  int exp_flags;               // experiment (SPECEDGE_ATTN_EXP): bit 0 = no MMAs for unit 1 in pair passes,
                               // bit 1 = plain softmax loop, bit 2 = full M-tiles only (timing; wrong tails)
};

#define TRACE(i)                                                                                  \
  do {                                                                                            \
    if (ta.trace && blockIdx.x == 0 && blockIdx.y == 0 && (i) < 1024) ta.trace[(i)] = clock64(); \
  } while (0)

template <int HD, int NQ>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQ2,
              const __grid_constant__ CUtensorMap tmQ4, const __grid_constant__ CUtensorMap tmPool,
              const __grid_constant__ CUtensorMap tmTree, const __grid_constant__ TcArgs ta) {
  pdl_begin();
  constexpr int KB = HD / 64;                       // 64-element hd blocks
  constexpr uint32_t QT_BYTES = 128 * HD * 2;       // one 128-row M-tile of Q
  constexpr uint32_t PG_BYTES = 64 * HD * 2;        // K (or V) of one 64-key sub-tile
  constexpr int NST = ring_stages(HD, NQ);
  const AttnArgs& a = ta.a;
  // 2 Q tiles + 5 K/V sub-tile stages = 224 KB of the 227 KB: the 1024-B alignment SW128 needs
  // comes from the dynamic-smem base itself (no static smem in this kernel); checked below.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sQ = smem_raw;                           // [2 units][KB][128 rows][128 B]
  uint8_t* sK = sQ + NQ * QT_BYTES;                 // [NST][KB][64 keys][128 B]
  uint8_t* sV = sK + NST * PG_BYTES;                // [NST][KB][64 keys][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + NST * PG_BYTES);
  uint64_t* q_full = bars;              // [1]
  uint64_t* q_empty = bars + 1;         // [1]
  uint64_t* kv_full = bars + 2;         // [NST]
  uint64_t* kv_empty = kv_full + NST;   // [NST]
  uint64_t* s_full = kv_empty + NST;    // [2 units][2 buffers]
  uint64_t* p_full = s_full + 4;        // [2][2]
  uint64_t* pv_done = p_full + 4;       // [2][2]
  uint64_t* o_full = pv_done + 4;       // [1]
  uint64_t* o_empty = o_full + 1;       // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);
  // completes once per pass whose epilogue merged replicas through the K/V ring: the producer
  // waits on it in order (it may run two passes ahead of o_empty, whose parity would alias)
  uint64_t* scr_done = o_empty + 2;
  float* s_ml = reinterpret_cast<float*>(o_empty + 3);          // [2 units][m, l][128 rows]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
  const int spm = ta.slots_per_mt;
  int* s_sched = reinterpret_cast<int*>(s_ml + 512);             // [4] balanced-mode cursor, [4] merge flag
  // ---- work items.  An item = (request r, kv head g, a range of the request's 64-key
  // sub-tiles: pages [p_begin, p_begin + npg) then tree halves [th0, th0 + ntree)), chunk c of
  // the nch chunks of (r, g).  Static mode: the item of blockIdx (x = r*KV + g, y = chunk of
  // pages_per_split pages, the tree in the request's last chunk).  Balanced mode (a.per_req == 2,
  // persistent grid): the (r, g) sub-tile sequences are concatenated (r-major, then g) into W
  // units and CTA b takes [b*Qw, (b+1)*Qw), Qw = max(ceil(W / grid), ceil(max_nsub / (n_splits -
  // 1))) so that no (r, g) is cut into more than n_splits chunks; the pipeline (K/V ring, TMEM
  // buffers, barrier phases) runs on across the CTA's items.
  auto S_of = [&](int rr) { return min(a.req_S[rr], a.max_rows / G); };
  auto nsub_of = [&](int rr) { return (a.req_L[rr] + 63) / 64 + (S_of(rr) > 64 ? 2 : 1); };
  const bool balanced = a.per_req == 2;
  // per-item state (set by next_item; the lambdas below read it by reference)
  int r = 0, g = 0, c_idx = 0, nch = 1, S = 0, L = 0, row0 = 0, h = 0, n_mt = 0, n_pass = 0, npages = 0;
  int p_begin = 0, npg = 0, th0 = 0, ntree = 0, nsub = 0;
  bool single = true;
  struct Cursor { int pos, end, r, base, Qw; };
  auto set_item = [&](int rr, int gg, int j0, int j1, int cc, int nc) {
    r = rr; g = gg; c_idx = cc; nch = nc;
    S = S_of(r); L = a.req_L[r]; row0 = a.req_row0[r]; h = a.req_h[r];
    n_mt = (S + spm - 1) / spm;
    if (ta.exp_flags & 4) n_mt = max(1, S / spm);   // experiment: full M-tiles only (no tail pass)
    // pass p: M-tiles 2p, 2p+1 ("pair") or the last one alone; with one Q tile (NQ = 1, chosen
    // when every request fits one M-tile) every pass is a single pass over M-tile p
    n_pass = NQ == 2 ? (n_mt + 1) / 2 : n_mt;
    npages = (L + 63) / 64;
    p_begin = j0;
    npg = max(0, min(j1, npages) - j0);
    th0 = max(j0, npages) - npages;
    ntree = max(0, j1 - max(j0, npages));
    nsub = npg + ntree;
    single = nch == 1;
  };
  auto cursor0 = [&]() -> Cursor {
    if (balanced) return Cursor{(int)blockIdx.x * s_sched[0], min(s_sched[1], (int)(blockIdx.x + 1) * s_sched[0]), s_sched[2],
                                s_sched[3], s_sched[0]};
    return Cursor{0, 1, 0, 0, 0};
  };
  auto next_item = [&](Cursor& cu) -> bool {
    if (!balanced) {
      if (cu.pos++ != 0) return false;
      const int rr = blockIdx.x / a.KV, gg = blockIdx.x % a.KV, sp = blockIdx.y;
      const int np_ = (a.req_L[rr] + 63) / 64;
      const int nc = a.per_req ? max(1, (np_ + a.pages_per_split - 1) / a.pages_per_split) : a.n_splits;
      if (sp >= nc) return false;
      const int j0 = sp * a.pages_per_split;
      const int j1 = sp == nc - 1 ? nsub_of(rr) : min(np_, j0 + a.pages_per_split);
      set_item(rr, gg, min(j0, np_), j1, sp, nc);
      return true;
    }
    if (cu.pos >= cu.end || cu.r >= a.B) return false;
    const int n = nsub_of(cu.r);
    const int gg = (cu.pos - cu.base) / n;
    const int o = cu.base + gg * n;
    const int j0 = cu.pos - o, j1 = min(n, cu.end - o);
    set_item(cu.r, gg, j0, j1, (int)blockIdx.x - o / cu.Qw, (o + n - 1) / cu.Qw - o / cu.Qw + 1);
    cu.pos = o + j1;
    if (cu.pos >= cu.base + a.KV * n) { cu.base += a.KV * n; ++cu.r; }
    return true;
  };
  if (balanced && warp == 0) {
    // W, max nsub, and the request holding this CTA's first unit (lane-parallel over requests)
    int W = 0, mx = 0;
    for (int q0 = 0; q0 < a.B; q0 += 32) {
      const int n = q0 + lane < a.B ? nsub_of(q0 + lane) : 0;
      W += n;
      mx = max(mx, n);
    }
    for (int o = 16; o > 0; o >>= 1) {
      W += __shfl_xor_sync(0xffffffffu, W, o);
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    W *= a.KV;
    const int Qw = max((W + (int)gridDim.x - 1) / (int)gridDim.x, (mx + a.n_splits - 2) / (a.n_splits - 1));
    const int start = (int)blockIdx.x * Qw;
    int base = 0, rs = a.B;
    for (int q0 = 0; q0 < a.B && rs == a.B; q0 += 32) {
      const int n = q0 + lane < a.B ? a.KV * nsub_of(q0 + lane) : 0;
      int incl = n;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int excl = incl - n;
      const unsigned hit = __ballot_sync(0xffffffffu, n > 0 && start >= base + excl && start < base + incl);
      if (hit) {
        const int l = __ffs(hit) - 1;
        rs = q0 + l;
        base += __shfl_sync(0xffffffffu, excl, l);
      } else {
        base += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == 0) {
      s_sched[0] = Qw;
      s_sched[1] = W;
      s_sched[2] = rs;
      s_sched[3] = base;
    }
  }
  // sub-tile visited at step j of pass p: odd passes walk backwards (tree first) so they start on
  // what the previous pass left in L2.  Returns 0..npg-1 for pages, npg + t for tree half th0 + t.
  auto sub_of = [&](int p, int j) { return (p & 1) ? nsub - 1 - j : j; };
  auto pair_pass = [&](int p) { return NQ == 2 && 2 * p + 1 < n_mt; };
  // unit u's k-th sub-tile in pass p: pair pass -> every sub-tile (unit u = M-tile 2p+u);
  // single pass -> the two units split the sub-tiles of one M-tile (unit u takes j = 2k+u)
  auto nsub_u = [&](int p, int u) { return pair_pass(p) ? nsub : (nsub - u + 1) / 2; };
  auto j_of = [&](int p, int u, int k) { return pair_pass(p) ? k : 2 * k + u; };
  // M-tile of unit u in pass p and its row replication: a tile of <= floor(32/G) slots is loaded
  // 4 times (one copy per TMEM lane quarter), <= floor(64/G) slots twice.  Replica r of a unit
  // sees only keys [r*64/Rf, (r+1)*64/Rf) of every sub-tile with its own running max / sum / O,
  // so a small tail tile (cfg2: 4 rows) spreads its softmax over all four SM sub-partitions
  // instead of doubling one of them; replicas are merged in the epilogue.
  auto mt_of = [&](int p, int u) { return pair_pass(p) ? 2 * p + u : (NQ == 2 ? 2 * p : p); };
  auto rep_of = [&](int p, int u) {
    const int slots = min(spm, S - mt_of(p, u) * spm);
    return slots <= 32 / G ? 4 : (slots <= 64 / G ? 2 : 1);
  };

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    tma_prefetch(&tmQ);
    tma_prefetch(&tmQ2);
    tma_prefetch(&tmQ4);
    tma_prefetch(&tmPool);
    tma_prefetch(&tmTree);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 2);   // one commit per MMA issuer
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 2);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_full, 2);
    mbar_init(o_empty, 256);
    mbar_init(scr_done, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // TMEM columns: unit u owns S buffers [256u, 256u+64) and [256u+64, 256u+128) (P aliases the
  // first 32 columns of its buffer) and the O accumulator [256u+128, 256u+128+HD)
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRACE(1000);
  // one 32-column chunk of an output row: normalised bf16 (+ optional fp32) when the KV is not
  // split, else the unnormalised fp32 partial (the combine kernel merges splits with m, l)
  auto store_out = [&](size_t rh, int col, const float (&ov)[32], float, float) {
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
      float4* dst = reinterpret_cast<float4*>(a.opart + ((size_t)c_idx * a.R * a.H + rh) * HD + col);
#pragma unroll
      for (int e = 0; e < 32; e += 4) dst[e / 4] = make_float4(ov[e], ov[e + 1], ov[e + 2], ov[e + 3]);
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------------------- TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0, gp = 0;   // gp: passes over all items (barrier phases)
      bool scratch = false;         // the last pass merges replicas through the ring (epilogue)
      uint32_t nscr = 0;            // scr_done completions consumed
      Cursor cu = cursor0();
      while (next_item(cu)) {
      TRACE(900);
      if (balanced && c_idx == 0) a.nch_tab[r * a.KV + g] = nch;   // for the combine kernel
      const int* pages = a.block_table + (size_t)h * a.max_pages_per_seq + p_begin;
      for (int p = 0; p < n_pass; ++p, ++gp) {
        // the pass's Q tiles, issued right after its first K/V sub-tile: the K/V stream (HBM) is
        // the long pole, Q (just written by the QKV GEMM) comes from L2
        auto issue_q = [&]() {
          const int nq = pair_pass(p) ? 2 : 1;
          mbar_wait(q_empty, (gp & 1) ^ 1);
          uint32_t qbytes = 0;
          for (int u = 0; u < nq; ++u) qbytes += (uint32_t)rep_of(p, u) * (128 / rep_of(p, u) / G) * G * 128 * KB;
          mbar_expect_tx(q_full, qbytes);
          for (int u = 0; u < nq; ++u) {
            const int rf = rep_of(p, u);
            const CUtensorMap* tq = rf == 4 ? &tmQ4 : (rf == 2 ? &tmQ2 : &tmQ);
            for (int rr = 0; rr < rf; ++rr)
              for (int kb = 0; kb < KB; ++kb)
                tma_load_3d(sQ + u * QT_BYTES + kb * 128 * 128 + rr * (128 / rf) * 128, tq, q_full, kb * 64, g * G,
                            row0 + mt_of(p, u) * spm);
          }
          if (gp == 0) TRACE(901);
        };
        // the previous pass's epilogue merged replicas through the K/V ring: no K/V load may land
        // in the ring before that merge is done (o_empty of that pass)
        if (scratch) mbar_wait(scr_done, nscr++ & 1);
        scratch = rep_of(p, 0) > 1 || (pair_pass(p) && rep_of(p, 1) > 1);
        int next_page = nsub > 0 && sub_of(p, 0) < npg ? __ldg(pages + sub_of(p, 0)) : 0;
        // L2 prefetch of the pages kPrefetch sub-tiles ahead of the ring: the ring holds only a few
        // sub-tiles in flight, so HBM latency would otherwise bound the per-SM stream rate
        auto prefetch = [&](int jj) {
          if (jj >= nsub) return;
          const int sjj = sub_of(p, jj);
          if (sjj >= npg) return;
          const int rk = (((a.layer * a.num_pages + __ldg(pages + sjj)) * 2 + 0) * a.KV + g) * 64;
          for (int kb = 0; kb < KB; ++kb) {
            tma_prefetch_l2_2d(&tmPool, kb * 64, rk);
            tma_prefetch_l2_2d(&tmPool, kb * 64, rk + a.KV * 64);
          }
        };
        if (gp == 0) TRACE(902);
        const int kPrefetch = ta.prefetch;
        for (int jj = 0; jj < kPrefetch; ++jj) prefetch(jj);
        for (int j = 0; j < nsub; ++j) {
          if (kPrefetch) prefetch(j + kPrefetch);
          const int sj = sub_of(p, j);
          const int page = next_page;   // page ids are read one sub-tile ahead of their use
          if (j + 1 < nsub && sub_of(p, j + 1) < npg) next_page = __ldg(pages + sub_of(p, j + 1));
          mbar_wait(&kv_empty[stage], phase ^ 1);
          mbar_expect_tx(&kv_full[stage], 2 * PG_BYTES);
          uint8_t* dk = sK + stage * PG_BYTES;
          uint8_t* dv = sV + stage * PG_BYTES;
          int rk, rv;
          const CUtensorMap* tm;
          if (sj < npg) {
            rk = (((a.layer * a.num_pages + page) * 2 + 0) * a.KV + g) * 64;
            rv = rk + a.KV * 64;
            tm = &tmPool;
          } else {
            const int th = th0 + sj - npg;
            rk = ((a.layer * 2 + 0) * a.KV + g) * a.R_cap + row0 + 64 * th;
            rv = ((a.layer * 2 + 1) * a.KV + g) * a.R_cap + row0 + 64 * th;
            tm = &tmTree;
          }
          for (int kb = 0; kb < KB; ++kb) {
            tma_load_2d(dk + kb * 64 * 128, tm, &kv_full[stage], kb * 64, rk);
            tma_load_2d(dv + kb * 64 * 128, tm, &kv_full[stage], kb * 64, rv);
          }
          if (gp == 0) TRACE(j);
          if (++stage == NST) { stage = 0; phase ^= 1; }
          if (j == 0) issue_q();
        }
        if (nsub == 0) issue_q();
      }
      }
    }
  } else if (warp == 1 || warp == kWarps - 1) {
    // ------------------------------------------------------------------------- MMA issuers
    // one issuing thread per unit (warp 1: unit 0, last warp: unit 1), so neither unit's QK/PV
    // issue waits behind the other's barriers; per unit the tcgen05 ops stay in program order.
    const int u = warp == 1 ? 0 : 1;
    if (elect_one()) {
      const uint32_t id_qk = idesc_f16(128, 64, false);
      const uint32_t id_pv = idesc_f16(128, HD, true);
      uint32_t sub_base = 0;           // sub-tiles streamed before this pass (ring position)
      uint32_t kc = 0;                 // this unit's sub-tiles consumed (all passes): buffer kc & 1
      uint32_t gp = 0;                 // passes over all items
      Cursor cu = cursor0();
      while (next_item(cu)) {
      for (int p = 0; p < n_pass; ++p, ++gp) {
        const bool pr = pair_pass(p);
        const int nk = nsub_u(p, u);
        if (gp == 0) TRACE(910 + u);
        mbar_wait(q_full, gp & 1);
        if (gp == 0) TRACE(912 + u);
        tc_fence_after();
        // QK of this unit's k-th sub-tile of the pass into S buffer (kc + k) & 1
        auto issue_qk = [&](int k) {
          const uint32_t gi = sub_base + (uint32_t)j_of(p, u, k);
          mbar_wait(&kv_full[gi % NST], (gi / NST) & 1);
          if (gp == 0 && k < 64) TRACE(640 + 64 * u + k);
          tc_fence_after();
          const uint32_t qaddr = smem_u32(sQ + (pr ? u : 0) * QT_BYTES);
          const uint32_t kaddr = smem_u32(sK + (gi % NST) * PG_BYTES);
          const uint32_t b = (kc + k) & 1;
          const uint32_t s_tm = tmem + u * 256 + b * 64;
          if (!((ta.exp_flags & 1) && pr && u == 1)) {
#pragma unroll
          for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc_mma_f16(s_tm, umma_desc_sw128(qaddr + kb * 16384 + kk * 32),
                         umma_desc_sw128(kaddr + kb * 8192 + kk * 32), id_qk, (kb | kk) != 0);
          }
          tc_commit(&s_full[u * 2 + b]);
          if (k == nk - 1) tc_commit(q_empty);   // last QK of the pass: Q may be reloaded
        };
        for (int k = 0; k < 2 && k < nk; ++k) issue_qk(k);
        if (gp == 0) TRACE(914 + u);
        if (nk == 0) tc_commit(q_empty);
        for (int k = 0; k < nk; ++k) {
          const uint32_t kg = kc + k;
          const uint32_t b = kg & 1;
          mbar_wait(&p_full[u * 2 + b], (kg >> 1) & 1);
          if (k == 0) mbar_wait(o_empty, (gp & 1) ^ 1);   // the previous pass's O has been drained
          tc_fence_after();
          const uint32_t gi = sub_base + (uint32_t)j_of(p, u, k);
          const uint32_t vaddr = smem_u32(sV + (gi % NST) * PG_BYTES);
          const uint32_t p_tm = tmem + u * 256 + b * 64;
          const uint32_t o_tm = tmem + u * 256 + 128;
          if (!((ta.exp_flags & 1) && pr && u == 1)) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {   // 16 keys (8 packed fp16 columns) per k-step
            const uint64_t bd = umma_desc_mn_sw128(vaddr + kk * 2048, 64 * 128);
            tc_mma_ts(o_tm, p_tm + kk * 8, bd, id_pv, (k | kk) != 0);
          }
          }
          tc_commit(&pv_done[u * 2 + b]);
          // kv_empty takes 2 arrivals per use: one per unit in a pair pass, both from the only
          // reader in a single pass
          tc_commit(&kv_empty[gi % NST]);
          if (!pr) tc_commit(&kv_empty[gi % NST]);
          // S buffer b takes sub-tile k+2 (in-order execution: after PV(k) has read P(k))
          if (k + 2 < nk) issue_qk(k + 2);
        }
        tc_commit(o_full);
        kc += nk;
        sub_base += nsub;
      }
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax + epilogue
    // warps 2..9: unit u = (warp-2)/4, one thread per TMEM lane (query row or a replica of one),
    // 64 keys per sub-tile.
    const int u = (warp - 2) >> 2;
    const int q = warp & 3;                   // TMEM lane quarter
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t s_base = tmem + u * 256 + lane_off;
    const uint32_t o_own = tmem + u * 256 + 128 + lane_off;
    const float sl2 = a.scale_log2;
    uint32_t kc = 0;   // this unit's sub-tiles consumed (all passes)
    uint32_t gp = 0;   // passes over all items
    Cursor cu = cursor0();
    while (next_item(cu)) {
    for (int p = 0; p < n_pass; ++p, ++gp) {
      const bool pr = pair_pass(p);
      const int mt = mt_of(p, u);
      const int rf = rep_of(p, u);
      const int rrows = 128 / rf;                       // lanes per replica
      const int rq = (q * 32) / rrows;                  // my replica
      const int ri = q * 32 + lane - rq * rrows;        // my row within the M-tile
      const int rows_mt = min(spm, S - mt * spm) * G;   // valid rows in this M-tile
      const bool valid_row = ri < rows_mt;
      const int slot = mt * spm + ri / G;
      const int j = ri % G;
      const uint64_t anc = (valid_row && slot > 0 && ntree > 0) ? __ldg(a.row_anc + row0 + slot) : 0ull;
      // my replica's key window within every 64-key sub-tile
      const uint64_t win = rf == 1 ? ~0ull : (((1ull << (64 / rf)) - 1ull) << (rq * (64 / rf)));
      const int nk = nsub_u(p, u);
      float m_used = -INFINITY, l = 0.f;
      // 64-bit visibility mask of sub-tile k's keys for my row
      auto key_mask = [&](int k) -> uint64_t {
        if (!valid_row) return 0ull;
        const int sj = sub_of(p, j_of(p, u, k));
        uint64_t mk;
        if (sj < npg) {
          const int kvalid = min(64, L - (p_begin + sj) * 64);
          mk = kvalid >= 64 ? ~0ull : ((1ull << kvalid) - 1ull);
        } else {
          // key 0 = root, key k >= 1 = node k-1: visible iff root or ancestor-or-self of my node
          const int th = th0 + sj - npg;
          const uint64_t lo = slot > 0 ? ((anc << 1) | 1ull) : 1ull;
          const uint64_t hi = slot > 0 ? (anc >> 63) : 0ull;
          const int n = S - 64 * th;   // tree keys in this half
          mk = (th ? hi : lo) & (n >= 64 ? ~0ull : ((1ull << n) - 1ull));
        }
        return mk & win;
      };
      // O *= alpha for the rows whose running max moved (warp-collective; PV(k-1) writes O and may
      // still be in flight -> wait for it first)
      auto rescale_o = [&](uint32_t kg, bool rescale, float alpha) {
        if (!__any_sync(0xffffffffu, rescale)) return;
        const uint32_t pb = (kg - 1) & 1;
        mbar_wait(&pv_done[u * 2 + pb], ((kg - 1) >> 1) & 1);
        tc_fence_after();
        // tcgen05.ld/st are warp-collective (.sync.aligned): the whole warp runs the loop, rows
        // without a rescale multiply by 1 (a per-lane branch here deadlocked the warp)
        const float f = rescale ? alpha : 1.f;
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t ov[32];
          tmem_ld_32x32b_x32(o_own + c * 32, ov);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * f);
          tmem_st_32x32b_x32(o_own + c * 32, ov);
        }
      };
      if (rf == 1 && !(ta.exp_flags & 2)) {
        // ---- unreplicated tile, software-pipelined: S(k+1) is loaded from TMEM while P(k) is
        // stored, and once a running max exists the exponentials start right away with it, the
        // sub-tile max being tracked alongside (only a row whose max grew by more than 8 redoes
        // its exponentials) — the same m_used sequence, hence the same bits, as the plain loop
        uint32_t sv[64];
        auto issue_ld = [&](int k, uint32_t (&dst)[64]) {
          const uint32_t kg = kc + k, b = kg & 1;
          mbar_wait(&s_full[u * 2 + b], (kg >> 1) & 1);
          tc_fence_after();
          tmem_ld_32x32b_x32(s_base + b * 64, *reinterpret_cast<uint32_t(*)[32]>(dst));
          tmem_ld_32x32b_x32(s_base + b * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(dst + 32));
        };
        auto step = [&](int k) {
          const uint32_t kg = kc + k, b = kg & 1;
          const uint32_t s_tm = s_base + b * 64;
          tmem_ld_wait();
          const uint64_t mk = key_mask(k);
          const bool any = __any_sync(0xffffffffu, mk != 0ull);
          const bool full = __all_sync(0xffffffffu, mk == ~0ull);
          float ls = 0.f;
          bool rescale = false;
          float alpha = 1.f;
          if (any) {
            const uint32_t mlo = (uint32_t)mk, mhi = (uint32_t)(mk >> 32);
            // P = 2^(s*scale - mb) as packed fp16 pairs (masked keys: -inf -> 0); returns the
            // row sum, mx_out = the masked sub-tile max (log2 domain)
            auto exps = [&](float mb, float& mx_out) {
              float m0 = -INFINITY, m1 = -INFINITY, ls0 = 0.f, ls1 = 0.f;
              if (full) {
#pragma unroll
                for (int e = 0; e < 64; e += 2) {
                  const float s0 = __uint_as_float(sv[e]), s1 = __uint_as_float(sv[e + 1]);
                  m0 = fmaxf(m0, s0);
                  m1 = fmaxf(m1, s1);
                  const float p0 = ex2f(fmaf(s0, sl2, -mb));
                  const float p1 = ex2f(fmaf(s1, sl2, -mb));
                  ls0 += p0;
                  ls1 += p1;
                  sv[e >> 1] = pack2(p0, p1);   // in place: sv[e], sv[e + 1] are consumed
                }
              } else {
#pragma unroll
                for (int e = 0; e < 64; e += 2) {
                  const uint32_t wd = e < 32 ? mlo : mhi;
                  const float s0 = ((wd >> (e & 31)) & 1u) ? __uint_as_float(sv[e]) : -INFINITY;
                  const float s1 = ((wd >> ((e + 1) & 31)) & 1u) ? __uint_as_float(sv[e + 1]) : -INFINITY;
                  m0 = fmaxf(m0, s0);
                  m1 = fmaxf(m1, s1);
                  const float p0 = ex2f(fmaf(s0, sl2, -mb));
                  const float p1 = ex2f(fmaf(s1, sl2, -mb));
                  ls0 += p0;
                  ls1 += p1;
                  sv[e >> 1] = pack2(p0, p1);
                }
              }
              mx_out = fmaxf(m0, m1) * sl2;
              return ls0 + ls1;
            };
            float mx;
            const bool first = m_used == -INFINITY;
            ls = exps(first ? 0.f : m_used, mx);
            // a row whose max grew by more than 8 (or its first visible keys) takes the new max:
            // reload S(k) from TMEM (still there) and redo the exponentials with it
            const bool redo = (mx > m_used + 8.f) || (first && mx > -INFINITY);
            if (__any_sync(0xffffffffu, redo)) {
              if (redo) {
                alpha = first ? 0.f : ex2f(m_used - mx);
                rescale = k > 0 && !first;
                l *= alpha;
                m_used = mx;
              }
              tmem_ld_32x32b_x32(s_tm, *reinterpret_cast<uint32_t(*)[32]>(sv));
              tmem_ld_32x32b_x32(s_tm + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
              tmem_ld_wait();
              float dummy;
              ls = exps(m_used == -INFINITY ? 0.f : m_used, dummy);
            }
            l += ls;
          }
          if (any) {   // P packed into sv[0, 32)
            tmem_st_32x32b_x16(s_tm, *reinterpret_cast<uint32_t(*)[16]>(sv));
            tmem_st_32x32b_x16(s_tm + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
          } else {
            uint32_t z[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) z[e] = 0u;
            tmem_st_32x32b_x16(s_tm, z);
            tmem_st_32x32b_x16(s_tm + 16, z);
          }
          if (any) rescale_o(kg, rescale, alpha);   // before PV(k) may add into O
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&p_full[u * 2 + b]);
          // S(k+1): its load is in flight while the loop comes around
          if (k + 1 < nk) issue_ld(k + 1, sv);
        };
        if (nk > 0) issue_ld(0, sv);
        for (int k = 0; k < nk; ++k) step(k);
      } else
      for (int k = 0; k < nk; ++k) {
        const uint32_t kg = kc + k;
        const uint32_t b = kg & 1;
        const uint32_t s_tm = s_base + b * 64;
        mbar_wait(&s_full[u * 2 + b], (kg >> 1) & 1);
        if (gp == 0 && lane == 0 && q == 0) TRACE(256 + 64 * u + k);
        tc_fence_after();
        const int sj = sub_of(p, j_of(p, u, k));
        // 64-bit visibility mask of the sub-tile's keys for my row
        uint64_t mk = 0ull;
        if (valid_row) {
          if (sj < npg) {
            const int kvalid = min(64, L - (p_begin + sj) * 64);
            mk = kvalid >= 64 ? ~0ull : ((1ull << kvalid) - 1ull);
          } else {
            // key 0 = root, key k >= 1 = node k-1: visible iff root or ancestor-or-self of my node
            const int th = th0 + sj - npg;
            const uint64_t lo = slot > 0 ? ((anc << 1) | 1ull) : 1ull;
            const uint64_t hi = slot > 0 ? (anc >> 63) : 0ull;
            const int n = S - 64 * th;   // tree keys in this half
            mk = (th ? hi : lo) & (n >= 64 ? ~0ull : ((1ull << n) - 1ull));
          }
          mk &= win;
        }
        const bool any = __any_sync(0xffffffffu, mk != 0ull);
        if (any) {
          // only my replica's key window [c0, c0 + W) is loaded, reduced and exponentiated; the
          // other P columns of the buffer are zeroed (they hold stale scores)
          auto body = [&](auto wc) {
            constexpr int W = decltype(wc)::value;
            const int c0 = W == 64 ? 0 : rq * W;
            const uint64_t mw = mk >> c0;   // bit e <-> key c0 + e
            const bool full = __all_sync(0xffffffffu, (W == 64 ? mk == ~0ull : (mw & ((1ull << W) - 1ull)) == ((1ull << W) - 1ull)));
            uint32_t sv[W];
            if constexpr (W == 16) {
              tmem_ld_32x32b_x16(s_tm + c0, *reinterpret_cast<uint32_t(*)[16]>(sv));
            } else {
#pragma unroll
              for (int h = 0; h < W / 32; ++h)
                tmem_ld_32x32b_x32(s_tm + c0 + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(sv + 32 * h));
            }
            tmem_ld_wait();
            if (gp == 0 && lane == 0 && q == 0 && k < 16) TRACE(512 + 64 * u + 4 * k);
            float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
            if (full) {
#pragma unroll
              for (int e = 0; e < W; e += 4) {
                m0 = fmaxf(m0, __uint_as_float(sv[e]));
                m1 = fmaxf(m1, __uint_as_float(sv[e + 1]));
                m2 = fmaxf(m2, __uint_as_float(sv[e + 2]));
                m3 = fmaxf(m3, __uint_as_float(sv[e + 3]));
              }
            } else {
              const uint32_t mlo = (uint32_t)mw, mhi = (uint32_t)(mw >> 32);
#pragma unroll
              for (int e = 0; e < W; e += 2) {
                const uint32_t wd = e < 32 ? mlo : mhi;
                m0 = fmaxf(m0, ((wd >> (e & 31)) & 1u) ? __uint_as_float(sv[e]) : -INFINITY);
                m1 = fmaxf(m1, ((wd >> ((e + 1) & 31)) & 1u) ? __uint_as_float(sv[e + 1]) : -INFINITY);
              }
            }
            const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * sl2;
            if (gp == 0 && lane == 0 && q == 0 && k < 16) TRACE(513 + 64 * u + 4 * k);
            float alpha = 1.f;
            bool rescale = false;
            if (mx > m_used + 8.f || (m_used == -INFINITY && mx > -INFINITY)) {
              alpha = m_used == -INFINITY ? 0.f : ex2f(m_used - mx);
              rescale = k > 0 && m_used != -INFINITY;
              l *= alpha;
              m_used = mx;
            }
            const float mb = m_used == -INFINITY ? 0.f : m_used;
            // P = 2^(s*scale - m) as packed fp16 pairs: keys c0 + e -> column (c0 + e) / 2
            float ls0 = 0.f, ls1 = 0.f;
            uint32_t pk[W / 2];
            if (full) {
#pragma unroll
              for (int e = 0; e < W; e += 2) {
                // kEmu8 of every 8 exponentials on the FMA pipe, the rest on MUFU
                const float x0 = fmaf(__uint_as_float(sv[e]), sl2, -mb);
                const float x1 = fmaf(__uint_as_float(sv[e + 1]), sl2, -mb);
                const float p0 = (e & 7) < kEmu8 ? exp2_fma(x0) : ex2f(x0);
                const float p1 = ((e + 1) & 7) < kEmu8 ? exp2_fma(x1) : ex2f(x1);
                ls0 += p0;
                ls1 += p1;
                pk[e >> 1] = pack2(p0, p1);
              }
            } else {
              const uint32_t mlo = (uint32_t)mw, mhi = (uint32_t)(mw >> 32);
#pragma unroll
              for (int e = 0; e < W; e += 2) {
                const uint32_t wd = e < 32 ? mlo : mhi;
                const float p0 = ((wd >> (e & 31)) & 1u) ? ex2f(fmaf(__uint_as_float(sv[e]), sl2, -mb)) : 0.f;
                const float p1 = ((wd >> ((e + 1) & 31)) & 1u) ? ex2f(fmaf(__uint_as_float(sv[e + 1]), sl2, -mb)) : 0.f;
                ls0 += p0;
                ls1 += p1;
                pk[e >> 1] = pack2(p0, p1);
              }
            }
            uint32_t z[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) z[e] = 0u;
            if constexpr (W == 64) {
              tmem_st_32x32b_x16(s_tm, *reinterpret_cast<uint32_t(*)[16]>(pk));
              tmem_st_32x32b_x16(s_tm + 16, *reinterpret_cast<uint32_t(*)[16]>(pk + 16));
            } else if constexpr (W == 32) {   // columns [16 rq, 16 rq + 16)
              tmem_st_32x32b_x16(s_tm + 16 * rq, *reinterpret_cast<uint32_t(*)[16]>(pk));
              tmem_st_32x32b_x16(s_tm + 16 * (rq ^ 1), z);
            } else {                          // columns [8 rq, 8 rq + 8)
#pragma unroll
              for (int c = 0; c < 4; ++c)
                tmem_st_32x32b_x8(s_tm + 8 * c, c == rq ? *reinterpret_cast<uint32_t(*)[8]>(pk)
                                                        : *reinterpret_cast<uint32_t(*)[8]>(z));
            }
            l += ls0 + ls1;
            if (gp == 0 && lane == 0 && q == 0 && k < 16) TRACE(514 + 64 * u + 4 * k);
            if (__any_sync(0xffffffffu, rescale)) {
              // O *= alpha: PV(k-1) writes O and may still be in flight -> wait for it
              const uint32_t pb = (kg - 1) & 1;
              mbar_wait(&pv_done[u * 2 + pb], ((kg - 1) >> 1) & 1);
              tc_fence_after();
              // tcgen05.ld/st are warp-collective (.sync.aligned): the whole warp runs the loop,
              // rows without a rescale multiply by 1 (a per-lane branch here deadlocked the warp)
              const float f = rescale ? alpha : 1.f;
#pragma unroll 1
              for (int c = 0; c < HD / 32; ++c) {
                uint32_t ov[32];
                tmem_ld_32x32b_x32(o_own + c * 32, ov);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * f);
                tmem_st_32x32b_x32(o_own + c * 32, ov);
              }
            }
          };
          if (rf == 1) body(std::integral_constant<int, 64>{});
          else if (rf == 2) body(std::integral_constant<int, 32>{});
          else body(std::integral_constant<int, 16>{});
        } else {
          // no visible key in this sub-tile for any row of this warp: P = 0
          uint32_t z[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) z[e] = 0u;
          tmem_st_32x32b_x16(s_tm, z);
          tmem_st_32x32b_x16(s_tm + 16, z);
        }
        tmem_st_wait();
        if (gp == 0 && lane == 0 && q == 0) TRACE(384 + 64 * u + k);
        tc_fence_before();
        mbar_arrive(&p_full[u * 2 + b]);
      }
      kc += nk;
      // ---- epilogue of the pass
      mbar_wait(o_full, gp & 1);
      tc_fence_after();
      const size_t rh = (size_t)(row0 + slot) * a.H + (size_t)g * G + j;
      const int rf_any = max(rep_of(p, 0), pr ? rep_of(p, 1) : 1);
      if (rf == 1) {
        s_ml[u * 256 + q * 32 + lane] = m_used;
        s_ml[u * 256 + 128 + q * 32 + lane] = l;
      }
      if (rf > 1) {
        // partial (m, l, O) of every replica -> the K/V ring, idle now: o_full says every MMA
        // reading the ring has completed, and the producer loads nothing into it before this
        // pass's scr_done
        // replica partial pidx = u*rf + rq occupies rows [pidx*rrows, (pidx+1)*rrows) of a
        // 256-row scratch (rf * rrows = 128 per unit): in a pair pass each unit merges its own
        // replicas, in a single pass both units' replicas of the one tile are merged together
        const int pidx = u * rf + rq;
        constexpr int PS = HD + 4;                        // padded row stride (floats)
        float* part = reinterpret_cast<float*>(sK);       // [256 rows][PS]
        float* pm = part + (size_t)256 * PS;              // [256 rows]
        float* pl = pm + 256;
        pm[pidx * rrows + ri] = m_used;
        pl[pidx * rrows + ri] = l;
        float* dst = part + ((size_t)pidx * rrows + ri) * PS;
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t ov[32];
          tmem_ld_32x32b_x32(o_own + c * 32, ov);
          tmem_ld_wait();
          if (valid_row && m_used != -INFINITY) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(dst + c * 32 + e) =
                  make_float4(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1]), __uint_as_float(ov[e + 2]),
                              __uint_as_float(ov[e + 3]));
          }
        }
      }
      named_bar_sync(2, 256);
      if (rf == 1) {
        float ms, lt, f0, f1;
        int c_lo, c_hi;
        const int rl = q * 32 + lane;
        if (pr) {   // my unit's own M-tile: all HD columns of my row
          ms = m_used;
          lt = l;
          f0 = 1.f;
          f1 = 0.f;
          c_lo = 0;
          c_hi = HD / 32;
        } else {    // both units hold partial (m, l, O) of the same rows: merge, unit u writes half
          const float ma = s_ml[rl], mbv = s_ml[256 + rl];
          ms = fmaxf(ma, mbv);
          f0 = ma == -INFINITY ? 0.f : ex2f(ma - ms);
          f1 = mbv == -INFINITY ? 0.f : ex2f(mbv - ms);
          lt = s_ml[128 + rl] * f0 + s_ml[384 + rl] * f1;
          c_lo = u * (HD / 64);
          c_hi = c_lo + HD / 64;
        }
        const float inv = single ? (lt > 0.f ? 1.f / lt : 0.f) : 1.f;
        f0 *= inv;
        f1 *= inv;
#pragma unroll 1
        for (int c = c_lo; c < c_hi; ++c) {
          const int col = c * 32;
          uint32_t oa[32];
          float ov[32];
          tmem_ld_32x32b_x32((pr ? o_own : tmem + 128 + lane_off) + col, oa);
          tmem_ld_wait();
          // a unit without any visible key (or without sub-tiles) has factor 0 and an O that
          // was never written: select instead of multiplying so stale TMEM cannot inject NaN
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = f0 != 0.f ? __uint_as_float(oa[e]) * f0 : 0.f;
          if (!pr) {
            tmem_ld_32x32b_x32(tmem + 384 + lane_off + col, oa);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = f1 != 0.f ? fmaf(__uint_as_float(oa[e]), f1, ov[e]) : ov[e];
          }
          if (valid_row) store_out(rh, col, ov, ms, lt);
        }
        if (valid_row && !single && (pr || u == 0)) {
          a.mpart[(size_t)c_idx * a.R * a.H + rh] = ms;
          a.lpart[(size_t)c_idx * a.R * a.H + rh] = lt;
        }
      } else {
        // merge the replicas: the unit's (pair pass) or both units' (single pass) threads
        // cooperate over (row, 32-column chunk) items of the tile
        const int np_ = pr ? rf : 2 * rf;          // partials to merge, from pidx p0
        const int p0 = pr ? u * rf : 0;
        constexpr int PS = HD + 4;
        const float* part = reinterpret_cast<const float*>(sK) + (size_t)p0 * rrows * PS;
        const float* pm = reinterpret_cast<const float*>(sK) + (size_t)256 * PS + p0 * rrows;
        const float* pl = pm + 256;
        const int nthr = pr ? 128 : 256;
        const int tid = pr ? q * 32 + lane : (u * 128 + q * 32 + lane);
        const int items = rows_mt * (HD / 32);
        for (int it = tid; it < items; it += nthr) {
          const int row = it / (HD / 32), col = (it % (HD / 32)) * 32;
          float ms = -INFINITY;
          for (int pp = 0; pp < np_; ++pp) ms = fmaxf(ms, pm[pp * rrows + row]);
          float lt = 0.f, ov[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = 0.f;
          for (int pp = 0; pp < np_; ++pp) {
            const float mp = pm[pp * rrows + row];
            if (mp == -INFINITY) continue;
            const float f = ex2f(mp - ms);
            lt += pl[pp * rrows + row] * f;
            const float* src = part + ((size_t)pp * rrows + row) * PS + col;
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              const float4 v = *reinterpret_cast<const float4*>(src + e);
              ov[e] = fmaf(v.x, f, ov[e]);
              ov[e + 1] = fmaf(v.y, f, ov[e + 1]);
              ov[e + 2] = fmaf(v.z, f, ov[e + 2]);
              ov[e + 3] = fmaf(v.w, f, ov[e + 3]);
            }
          }
          const float inv = single ? (lt > 0.f ? 1.f / lt : 0.f) : 1.f;
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] *= inv;
          const int rslot = mt * spm + row / G;
          const size_t rrh = (size_t)(row0 + rslot) * a.H + (size_t)g * G + row % G;
          store_out(rrh, col, ov, ms, lt);
          if (!single && col == 0) {
            a.mpart[(size_t)c_idx * a.R * a.H + rrh] = ms;
            a.lpart[(size_t)c_idx * a.R * a.H + rrh] = lt;
          }
        }
      }
      (void)rf_any;
      tc_fence_before();
      mbar_arrive(o_empty);
      if (rep_of(p, 0) > 1 || (pr && rep_of(p, 1) > 1)) mbar_arrive(scr_done);
      named_bar_sync(2, 256);   // s_ml / ring reuse by the next pass
      if (balanced && a.merge_cnt && !single && p == n_pass - 1) {
        // the last CTA to finish a chunk of (r, g) merges all its chunks (split-KV combine, from
        // L2): the classic fence / counter / last-arriver pattern, no CTA ever waits on another
        const int et = (warp - 2) * 32 + lane;   // 0..255
        __threadfence();
        named_bar_sync(2, 256);
        if (et == 0) {
          int* cnt = a.merge_cnt + r * a.KV + g;
          const int prev = atomicAdd(cnt, 1);
          s_sched[4] = prev == nch - 1;
          if (prev == nch - 1) *cnt = 0;   // ready for the next launch
        }
        named_bar_sync(2, 256);
        if (s_sched[4]) {
          __threadfence();
          const size_t RH = (size_t)a.R * a.H;
          const int nrow = S * G;
          for (int idx = et; idx < nrow * (HD / 4); idx += 256) {
            const int rl = idx / (HD / 4), d = (idx % (HD / 4)) * 4;
            const size_t rh = (size_t)(row0 + rl / G) * a.H + (size_t)g * G + rl % G;
            float mv[8], lv[8];
            float mx = -INFINITY;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              mv[c] = c < nch ? __ldcg(a.mpart + c * RH + rh) : -INFINITY;
              lv[c] = c < nch ? __ldcg(a.lpart + c * RH + rh) : 0.f;
              mx = fmaxf(mx, mv[c]);
            }
            float lt = 0.f;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              if (mv[c] == -INFINITY) continue;
              const float w = ex2f(mv[c] - mx);
              lt += w * lv[c];
              const float4 v = __ldcg(reinterpret_cast<const float4*>(a.opart + (c * RH + rh) * HD + d));
              acc.x = fmaf(w, v.x, acc.x);
              acc.y = fmaf(w, v.y, acc.y);
              acc.z = fmaf(w, v.z, acc.z);
              acc.w = fmaf(w, v.w, acc.w);
            }
            const float inv = lt > 0.f ? 1.f / lt : 0.f;
            if (ta.O)
              *reinterpret_cast<uint2*>(ta.O + rh * HD + d) =
                  make_uint2(pack2_bf16(acc.x * inv, acc.y * inv), pack2_bf16(acc.z * inv, acc.w * inv));
            if (ta.O_f32)
              *reinterpret_cast<float4*>(ta.O_f32 + rh * HD + d) =
                  make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
          }
        }
        named_bar_sync(2, 256);   // s_sched[4] reuse
      }
    }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) TRACE(1001);
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

// Slots per 128-row M-tile: floor(128/G), or floor(64/G) with SPECEDGE_ATTN_HALF_TILES=1 (every
// full tile then runs with 2-way row replication, i.e. half the keys per softmax thread, at the
// price of more passes over the KV stream)
int attn_slots_per_tile(int G) {
  static const bool half = getenv("SPECEDGE_ATTN_HALF_TILES") && getenv("SPECEDGE_ATTN_HALF_TILES")[0] == '1';
  return (half && G <= 64) ? 64 / G : 128 / G;
}

template <int HD, int NQ>
cudaError_t launch_tc(const AttnArgs& a, int B, bf16* O, float* O_f32, cudaStream_t st) {
  CUtensorMap tq, tp, tt;
  const int spm = attn_slots_per_tile(a.G);
  const uint64_t pool_rows = (uint64_t)(a.layer + 1) * a.num_pages * 2 * a.KV * 64;
  const uint64_t tree_rows = (uint64_t)(a.layer + 1) * 2 * a.KV * a.R_cap;
  // replicated loads of small tail tiles: boxes of floor(64/G) / floor(32/G) slots (a tile is
  // replicated only when it fits its box; the max(1, .) maps are valid but unused)
  CUtensorMap tq2, tq4;
  if (!encode_fn() || !tmap_q(&tq, a.Q, (uint64_t)a.R, a.H, HD, a.G, spm) || !tmap_rows(&tp, a.pool, pool_rows, HD) ||
      !tmap_rows(&tt, a.tree_kv, tree_rows, HD))
    return cudaErrorInvalidValue;
  if (!tmap_q(&tq2, a.Q, (uint64_t)a.R, a.H, HD, a.G, std::max(1, 64 / a.G)) ||
      !tmap_q(&tq4, a.Q, (uint64_t)a.R, a.H, HD, a.G, std::max(1, 32 / a.G)))
    return cudaErrorInvalidValue;
  static const int pf = getenv("SPECEDGE_ATTN_PREFETCH") ? atoi(getenv("SPECEDGE_ATTN_PREFETCH")) : kPrefetchDefault;
  static unsigned long long* trace = nullptr;
  if (getenv("SPECEDGE_ATTN_TRACE") && !trace) cudaMalloc(&trace, 1024 * 8);
  static const int exp_flags = getenv("SPECEDGE_ATTN_EXP") ? atoi(getenv("SPECEDGE_ATTN_EXP")) : 0;
  TcArgs ta{a, O, O_f32, spm, pf, trace, exp_flags};
  if (trace) cudaMemsetAsync(trace, 0, 1024 * 8, st);
  constexpr int NST = ring_stages(HD, NQ);
  const size_t smem = (size_t)NQ * 128 * HD * 2 + (size_t)NST * 2 * 64 * HD * 2 + 8 * (18 + 2 * NST) + 512 * 4 + 32;
  static_assert((size_t)NQ * 128 * HD * 2 + (size_t)NST * 2 * 64 * HD * 2 + 8 * (18 + 2 * NST) + 512 * 4 + 32 <=
                    (size_t)kSmemMax, "attention smem");
  static PerDeviceOnce attr;   // per-device attribute
  if (attr.first()) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_tc<HD, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
    if (e != cudaSuccess) {
      attr.done.fetch_and(~(1ull << current_device()));
      return e;
    }
  }
  const dim3 grid = a.per_req == 2 ? dim3(a.grid_ctas) : dim3(B * a.KV, a.n_splits);
  {
    const cudaError_t le = launch_k(k_attn_tc<HD, NQ>, grid, dim3(kThreads), smem, st, tq, tq2, tq4, tp, tt, ta);
    if (le != cudaSuccess) return le;
  }
  if (trace) {
    static int calls = 0;
    if (++calls % 32 == 7) {
      static unsigned long long hb[1024];
      cudaStreamSynchronize(st);
      cudaMemcpy(hb, trace, sizeof(hb), cudaMemcpyDeviceToHost);
      const unsigned long long t0 = hb[1000];
      auto d = [&](int i) { return hb[i] ? (long long)(hb[i] - t0) : -1LL; };
      fprintf(stderr, "attn trace CTA0: end=%lld item=%lld qissued=%lld page=%lld | mma u0: pre_q=%lld q=%lld qk01=%lld u1: pre_q=%lld q=%lld qk01=%lld\n",
              d(1001), d(900), d(901), d(902), d(910), d(912), d(914), d(911), d(913), d(915));
      for (int k = 0; k < 16; ++k)
        fprintf(stderr, " k%2d PIPE u0: load=%6lld kv=%6lld s=%6lld p=%6lld || u1: load=%6lld kv=%6lld s=%6lld p=%6lld\n", k,
                d(2 * k), d(640 + k), d(256 + k), d(384 + k), d(2 * k + 1), d(704 + k), d(320 + k), d(448 + k));
      for (int k = 0; k < 16; ++k)
        fprintf(stderr, " k%2d SOFTMAX u0: s=%6lld ld=%6lld max=%6lld exp=%6lld p=%6lld || u1: s=%6lld ld=%6lld max=%6lld exp=%6lld p=%6lld\n",
                k, d(256 + k), d(512 + 4 * k), d(513 + 4 * k), d(514 + 4 * k), d(384 + k), d(320 + k), d(576 + 4 * k),
                d(577 + 4 * k), d(578 + 4 * k), d(448 + k));
    }
  }
  return cudaGetLastError();
}

}  // namespace

bool attention_tc_supported(int hd, int G) { return (hd == 64 || hd == 128) && G >= 1 && G <= 128; }

cudaError_t attention_tc_launch(const AttnArgs& a, int B, bf16* O, float* O_f32, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  // one Q tile (and a deeper K/V ring) when every request's rows fit one M-tile
  static const int force_nq = getenv("SPECEDGE_ATTN_NQ") ? atoi(getenv("SPECEDGE_ATTN_NQ")) : 0;
  const bool one = force_nq ? force_nq == 1 : a.max_rows / a.G <= attn_slots_per_tile(a.G);
  if (a.hd == 128) return one ? launch_tc<128, 1>(a, B, O, O_f32, st) : launch_tc<128, 2>(a, B, O, O_f32, st);
  if (a.hd == 64) return one ? launch_tc<64, 1>(a, B, O, O_f32, st) : launch_tc<64, 2>(a, B, O, O_f32, st);
  return cudaErrorInvalidValue;
}

}  // namespace se
