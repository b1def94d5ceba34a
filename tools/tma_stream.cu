// TMA streaming microbenchmark for the paged-KV access pattern of the tree attention: one CTA per
// SM, one producer thread loading random 16 KB pages (64 rows x 256 B = two 64x64 fp16 SW128
// boxes) into an N-slot ring, one consumer thread releasing every slot as soon as it is full
// (hold = H spin cycles).  Reports chip bandwidth for each (N, H); DRAM-resident (8 GB) and
// L2-resident (32 MB) buffers.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_2505_17052_b200/csrc/common.cuh"

using namespace se;

__global__ void __launch_bounds__(96, 1) k_stream(const __grid_constant__ CUtensorMap tm, const int* __restrict__ pages,
                                                   int n_pages_per_cta, int nslots, int hold, int ncons, int slot_kb, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int SB = slot_kb * 1024;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nslots * SB);
  uint64_t* empty = full + nslots;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int* pg = pages + (size_t)blockIdx.x * n_pages_per_cta;
  if (threadIdx.x == 0) {
    for (int j = 0; j < n_pages_per_cta; ++j) {
      const int s = j % nslots;
      mbar_wait(&empty[s], ((j / nslots) & 1) ^ 1);
      mbar_expect_tx(&full[s], SB);
      for (int h = 0; h < slot_kb / 16; ++h) {   // 16 KB K page (+ a second 16 KB page as V)
        const int row = pg[(j * (slot_kb / 16) + h) % n_pages_per_cta] * 64;
        tma_load_2d(smem + s * SB + h * 16384, &tm, &full[s], 0, row);
        tma_load_2d(smem + s * SB + h * 16384 + 8192, &tm, &full[s], 64, row);
      }
    }
  } else if (threadIdx.x == 32 || (threadIdx.x == 64 && ncons == 2)) {
    unsigned long long acc = 0;
    for (int j = threadIdx.x == 64 ? 1 : 0; j < n_pages_per_cta; j += ncons) {
      const int s = j % nslots;
      mbar_wait(&full[s], (j / nslots) & 1);
      acc += smem[s * SB + (j & 1023)];
      if (hold) {
        const long long t0 = clock64();
        while (clock64() - t0 < hold) {}
      }
      mbar_arrive(&empty[s]);
    }
    if (acc == 12345) sink[0] = acc;
  }
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  const size_t big = (size_t)8 << 30;
  void* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 0, big);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t bytes : {big, (size_t)32 << 20}) {
    const uint64_t rows = bytes / 256;
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    ((PFN)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int n_pages = (int)(rows / 64);
    const int per_cta = 2048;
    std::vector<int> pages((size_t)148 * per_cta);
    std::mt19937 rng(1);
    for (auto& p : pages) p = rng() % n_pages;
    int* pd;
    cudaMalloc(&pd, pages.size() * 4);
    cudaMemcpy(pd, pages.data(), pages.size() * 4, cudaMemcpyHostToDevice);
    struct Cfg { int ncons, slot_kb, hold; };
    for (Cfg c : {Cfg{1, 16, 0}, Cfg{1, 32, 0}, Cfg{2, 32, 1000}, Cfg{2, 32, 2300}, Cfg{2, 32, 3000}}) {
      for (int ns : {2, 4, 5, 6}) {
        const size_t smem = (size_t)ns * c.slot_kb * 1024 + 2 * ns * 8;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        k_stream<<<148, 96, smem>>>(tm, pd, per_cta, ns, c.hold, c.ncons, c.slot_kb, sink);
        cudaEventRecord(e0);
        k_stream<<<148, 96, smem>>>(tm, pd, per_cta, ns, c.hold, c.ncons, c.slot_kb, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s cons %d hold %4d slots %2d x %2d KB: %6.0f GB/s  %s\n", bytes == big ? "HBM" : "L2 ", c.ncons, c.hold,
               ns, c.slot_kb, 148.0 * per_cta * c.slot_kb * 1024 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
      }
    }
    cudaFree(pd);
  }
  return 0;
}
