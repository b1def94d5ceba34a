// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M = 128) issue-to-completion rate as a
// function of N, for A from shared memory (SS) and A from TMEM (TS), on one SM.  Operand values
// are irrelevant (zero-filled smem).  Build + run (GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_17052_b200/csrc \
//        tools/mma_rate.cu -o /tmp/mma_rate && /tmp/mma_rate
#include "common.cuh"

#include <cstdio>

using namespace se;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int NACC>
__global__ void k_rate(int N, int ts, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;               // 128 x 64 fp16, SW128 (16 KB)
  uint8_t* B = sm + 16384;       // 256 x 64 fp16 (32 KB)
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t ad = umma_desc_sw128(smem_u32(A));
    const uint64_t bd = umma_desc_sw128(smem_u32(B));
    // warm-up
    for (int i = 0; i < 8; ++i) tc_mma_f16(tmem, ad, bd, idesc, 1);
    tc_commit(&bar);
    while (!mbar_try_wait(&bar, 0)) {}
    const long long t0 = clock64();
    // NACC independent accumulators (D = columns [a * N, ...)), A from TMEM at col 384;
    // 8-way unrolled straight-line issue
    if (ts) {
      for (int i = 0; i < reps; i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ts(tmem + (uint32_t)((k % NACC) * N), tmem + 384, bd, idesc, 1);
      }
    } else {
      for (int i = 0; i < reps; i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) tc_mma_f16(tmem + (uint32_t)((k % NACC) * N), ad, bd, idesc, 1);
      }
    }
    const long long t1 = clock64();
    tc_commit(&bar);
    while (!mbar_try_wait(&bar, 1)) {}
    const long long t2 = clock64();
    out[0] = t1 - t0;   // issue time
    out[1] = t2 - t0;   // completion time
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// Latency of a short dependent group (the attention's per-sub-tile chains): n MMAs into one
// accumulator, commit, wait -> cycles from the first issue to the mbarrier completing
__global__ void k_lat(int N, int ts, int n, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;
  uint8_t* B = sm + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t ad = umma_desc_sw128(smem_u32(A));
    const uint64_t bd = umma_desc_sw128(smem_u32(B));
    uint32_t ph = 0;
    long long best = 1LL << 60;
    for (int rep = 0; rep < 16; ++rep) {
      const long long t0 = clock64();
      for (int k = 0; k < n; ++k) {
        if (ts) mma_ts(tmem, tmem + 384, bd, idesc, k > 0);
        else tc_mma_f16(tmem, ad, bd, idesc, k > 0);
      }
      tc_commit(&bar);
      while (!mbar_try_wait(&bar, ph)) {}
      ph ^= 1;
      const long long t1 = clock64();
      if (rep > 2 && t1 - t0 < best) best = t1 - t0;
    }
    out[0] = best;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  {
    long long* dl;
    cudaMalloc(&dl, 8);
    cudaFuncSetAttribute(k_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int ts = 0; ts < 2; ++ts)
      for (int N : {64, 128})
        for (int n : {1, 4, 8}) {
          k_lat<<<1, 128, 64 * 1024>>>(N, ts, n, dl);
          long long h;
          cudaMemcpy(&h, dl, 8, cudaMemcpyDeviceToHost);
          printf("latency %s M=128 N=%3d: %d dependent MMAs -> %lld cycles issue-to-complete\n", ts ? "TS" : "SS", N, n, h);
        }
  }
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k_rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_rate<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_rate<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int reps = 4096;
  for (int ts = 0; ts < 2; ++ts)
    for (int N : {16, 32, 64, 128, 256})
      for (int nacc : {1, 2, 4}) {
        if (nacc * N > 384) continue;
        if (nacc == 1) k_rate<1><<<1, 128, 64 * 1024>>>(N, ts, reps, d);
        if (nacc == 2) k_rate<2><<<1, 128, 64 * 1024>>>(N, ts, reps, d);
        if (nacc == 4) k_rate<4><<<1, 128, 64 * 1024>>>(N, ts, reps, d);
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const double cyc = (double)h[1] / reps;
        const double macs = 128.0 * N * 16;
        printf("%s M=128 N=%3d K=16 acc=%d: %.1f cycles/instr (issue %.1f), %.0f MAC/clk/SM\n", ts ? "TS" : "SS", N,
               nacc, cyc, (double)h[0] / reps, macs / cyc);
      }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
