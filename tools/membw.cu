// DRAM read bandwidth for chunked random access: every chunk of C bytes is contiguous, chunks are
// visited in a random permutation (the paged-KV pattern: one page of one kv head = 16 KB at hd
// 128).  Also a sequential read for reference.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void k_read(const uint4* __restrict__ buf, const int* __restrict__ perm, int n_chunks, int chunk_u4,
                       unsigned long long* out) {
  uint32_t acc = 0;
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const uint4* p = buf + (size_t)perm[c] * chunk_u4;
#pragma unroll 4
    for (int i = threadIdx.x; i < chunk_u4; i += blockDim.x) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t total = (size_t)8 << 30;
  uint4* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* out;
  cudaMalloc(&out, 8);
  int* perm_d;
  cudaMalloc(&perm_d, (total / 4096) * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sizes[] = {4096, 8192, 16384, 32768, 65536, 262144};
  for (int seq = 0; seq < 2; ++seq)
    for (int cs : sizes) {
      const int n = (int)(total / cs);
      std::vector<int> perm(n);
      for (int i = 0; i < n; ++i) perm[i] = i;
      if (!seq) std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
      cudaMemcpy(perm_d, perm.data(), n * 4, cudaMemcpyHostToDevice);
      for (int threads : {256, 1024}) {
        for (int it = 0; it < 2; ++it) k_read<<<148 * (2048 / threads), threads>>>(buf, perm_d, n, cs / 16, out);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int it = 0; it < reps; ++it) k_read<<<148 * (2048 / threads), threads>>>(buf, perm_d, n, cs / 16, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s chunk %7d B threads %4d: %.0f GB/s\n", seq ? "seq " : "rand", cs, threads, total * reps / (ms * 1e6));
      }
    }
  return 0;
}
