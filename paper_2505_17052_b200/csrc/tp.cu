// Tensor parallelism for the verify step (SURVEY §8(a) a12, §8(e) "Tensor parallel TP = 8"):
// head-parallel attention, column-parallel QKV / gate-up, row-parallel O / down followed by a
// sum all-reduce of the fp32 [R, d] residual update (C1, C2), vocab-parallel LM head followed by
// an all-gather of the per-row (score, id) winners (C3) and a replicated final argmax.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, the copy torch has already loaded when it
// is in the process), so libspecedge.so has no link-time NCCL dependency and TP = 1 never touches
// it.  All collectives are enqueued on the verify stream; every rank issues them in the same order.
#include "common.cuh"
#include "internal.h"

#include <dlfcn.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace se {

namespace {

struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  if (!h) return api;
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
  api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(dlsym(h, "ncclReduceScatter"));
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
           api.ReduceScatter;
  return api;
}

// C3 reduction: per row, the best (score, id) over the tp_size vocab shards; ties -> lowest id
// (amb. A7).  g = [tp][R][2] floats, id stored as int bits.
__global__ void k_tp_argmax(const float* __restrict__ g, int tp, int R, int* __restrict__ y, float* __restrict__ score,
                            int* __restrict__ row_target, float* __restrict__ row_score) {
  pdl_begin();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= R) return;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int k = 0; k < tp; ++k) {
    const float v = g[((size_t)k * R + row) * 2];
    const int i = __float_as_int(g[((size_t)k * R + row) * 2 + 1]);
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
  y[row] = bi;
  score[row] = best;
  if (row_target) row_target[row] = bi;
  if (row_score) row_score[row] = best;
}

__global__ void k_tp_pack(const int* __restrict__ y, const float* __restrict__ score, int R, float* __restrict__ out) {
  pdl_begin();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= R) return;
  out[2 * row] = score[row];
  out[2 * row + 1] = __int_as_float(y[row]);
}

}  // namespace

bool tp_available() { return nccl().ok; }

int tp_unique_id(uint8_t* out128) {
  NcclApi& n = nccl();
  if (!n.ok) return -1;
  ncclUniqueId id;
  if (n.GetUniqueId(&id) != ncclSuccess) return -2;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, 128);
  return 0;
}

int tp_comm_init(void** comm, const uint8_t* id128, int rank, int size) {
  NcclApi& n = nccl();
  if (!n.ok) return -1;
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  ncclComm_t c = nullptr;
  if (n.CommInitRank(&c, size, id, rank) != ncclSuccess) return -2;
  *comm = c;
  return 0;
}

void tp_comm_destroy(void* comm) {
  if (comm && nccl().ok) nccl().CommDestroy(reinterpret_cast<ncclComm_t>(comm));
}

// C1 / C2: in-place fp32 sum of the [R, d] residual updates of all ranks
cudaError_t tp_allreduce_f32(float* buf, size_t n, void* comm, cudaStream_t st) {
  if (nccl().AllReduce(buf, buf, n, ncclFloat32, ncclSum, reinterpret_cast<ncclComm_t>(comm), st) != ncclSuccess)
    return cudaErrorUnknown;
  return cudaSuccess;
}

// C1 / C2 as reduce-scatter + all-gather (row-sharded residual stream): in place, rank k's chunk
// of `per_rank` elements at buf + k * per_rank
cudaError_t tp_reduce_scatter_f32(float* buf, size_t per_rank, int rank, void* comm, cudaStream_t st) {
  if (nccl().ReduceScatter(buf, buf + (size_t)rank * per_rank, per_rank, ncclFloat32, ncclSum,
                           reinterpret_cast<ncclComm_t>(comm), st) != ncclSuccess)
    return cudaErrorUnknown;
  return cudaSuccess;
}
cudaError_t tp_all_gather_bf16(bf16* buf, size_t per_rank, int rank, void* comm, cudaStream_t st) {
  if (nccl().AllGather(buf + (size_t)rank * per_rank, buf, per_rank, ncclBfloat16, reinterpret_cast<ncclComm_t>(comm),
                       st) != ncclSuccess)
    return cudaErrorUnknown;
  return cudaSuccess;
}

// C3: gather every rank's per-row winner and reduce to the global target token
cudaError_t tp_argmax_gather(int* y, float* score, int R, float* gather, int tp, void* comm, int* row_target,
                             float* row_score, cudaStream_t st, int* launches) {
  float* mine = gather + (size_t)tp * R * 2;   // staging after the gather area
  {
    cudaError_t le = launch_k(k_tp_pack, dim3((R + 127) / 128), dim3(128), 0, st, y, score, R, mine);
    if (le != cudaSuccess) return le;
  }
  if (launches) *launches += 2;
  if (nccl().AllGather(mine, gather, (size_t)R * 2, ncclFloat32, reinterpret_cast<ncclComm_t>(comm), st) !=
      ncclSuccess)
    return cudaErrorUnknown;
  {
    cudaError_t le = launch_k(k_tp_argmax, dim3((R + 127) / 128), dim3(128), 0, st, (const float*)gather, tp, R, y, score, row_target, row_score);
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}



// ---------------------------------------------------------------------------------------------
// NEXT-F4: the reduce-scatter of the row-parallel GEMMs (O, down) fused over NVLink peer memory
// (SURVEY §8(f) rank 5).  Each rank owns an exchange buffer that all peers have mapped (CUDA IPC).
//   push (default): the GEMM epilogue stages every 32-row chunk of its fp32 partial in shared
//     memory and one lane per warp bulk-copies 8 of the 512-byte row segments (cp.async.bulk)
//     into the receive slot [src] of the rank that owns the row (sequence-parallel residual: rank
//     k owns rows [k*Rl, (k+1)*Rl)); the transfer rides on the GEMM, tile by tile.
//   pull (SPECEDGE_TP_F4=pull): the GEMM writes its partial locally; the owner's RMSNorm loads its
//     rows from every rank's buffer (NVLink loads for the peers').
// Either way the owner's RMSNorm sums the tp partials in rank order together with the residual
// add and the normalisation (deterministic), with no reduce-scatter kernel and no staging copy.
// (A first push version stored 4-byte lanes straight from registers to the peer; it stalled the
// epilogue.)  Measured on cfg4 TP=2 (profiles/README.md): push 800.8 vs NCCL 761.4 tok/s on one
// box (+5.2 %); pull ~ NCCL (its NVLink loads lengthen the RMSNorms by about what NCCL costs).
//
// Ordering: after the GEMM, k_tp_signal (one thread per peer) publishes an epoch with a
// system-scope release store into every peer's flag word [src]; before the RMSNorm, k_tp_wait
// spins with acquire loads until every peer's flag holds that epoch (bounded: traps after ~20 s
// rather than hang).  pull: one buffer suffices — a rank overwrites it (its next row-parallel
// GEMM) only after the bf16 all-gather that follows every peer's RMSNorm.  push: two receive
// buffers alternate per collective — a rank writes buffer b for op n+2 only after consuming op
// n+1, which every peer sent after consuming op n from b.
// ---------------------------------------------------------------------------------------------
namespace {

__global__ void k_tp_signal(unsigned long long* const* __restrict__ peer_flags, int tp, int rank,
                            unsigned long long epoch) {
  const int p = threadIdx.x;
  __threadfence_system();
  if (p < tp) {
    unsigned long long* f = peer_flags[p] + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
  }
}

__global__ void k_tp_wait(const unsigned long long* __restrict__ my_flags, int tp, unsigned long long epoch) {
  const int p = threadIdx.x;
  if (p < tp) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + p) : "memory");
      if (v >= epoch) break;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) __trap();   // a peer never arrived: fail, do not hang the GPU
      __nanosleep(64);
    }
  }
  __syncthreads();
}

}  // namespace

cudaError_t tp_fused_signal(specedge_model* m, cudaStream_t st, int* launches) {
  ++m->tp_epoch;
  if (launches) ++*launches;
  k_tp_signal<<<1, 32, 0, st>>>(m->tp_peer_flags_dev, m->tp_size, m->tp_rank, m->tp_epoch);
  return cudaGetLastError();
}

cudaError_t tp_fused_wait(specedge_model* m, cudaStream_t st, int* launches) {
  if (launches) ++*launches;
  k_tp_wait<<<1, 32, 0, st>>>(m->tp_flags, m->tp_size, m->tp_epoch);
  return cudaGetLastError();
}

// Collective (every rank, same arguments): receive buffers for up to max_rows rows, IPC handles
// exchanged with an NCCL all-gather, peers' buffers and flag words mapped.
int tp_fused_enable(specedge_model* m, int max_rows, cudaStream_t st) {
  const int tp = m->tp_size;
  if (tp < 2 || tp > kMaxFusedTp || max_rows <= 0 || !m->nccl) return -1;
  if (m->tp_fused_rows >= max_rows) return 0;
  if (m->tp_fused_rows) return -2;   // already enabled with a smaller capacity: not resizable
  // pull: [max_rows][d] fp32; push: [2][tp][Rl][d] — the larger of the two layouts
  const size_t Rl = ((size_t)max_rows + tp - 1) / tp;
  m->tp_fused_slot = Rl * m->cfg.d;
  const size_t part_bytes = (std::max((size_t)max_rows * m->cfg.d, 2 * (size_t)tp * m->tp_fused_slot) * 4 + 255) / 256 * 256;
  const size_t hn_bytes = ((size_t)max_rows * m->cfg.d * 2 + 255) / 256 * 256;   // all-gathered bf16 rows
  const size_t out_bytes = part_bytes + hn_bytes;
  const size_t bytes = out_bytes + 256;
  char* base = nullptr;
  if (cudaMalloc(&base, bytes) != cudaSuccess) return -3;
  m->allocs.push_back(base);
  cudaMemset(base, 0, bytes);
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, base) != cudaSuccess) return -4;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle");
  char* dh = nullptr;
  if (cudaMalloc(&dh, 64 * (size_t)tp) != cudaSuccess) return -3;
  cudaMemcpy(dh + 64 * (size_t)m->tp_rank, &h, 64, cudaMemcpyHostToDevice);
  if (nccl().AllGather(dh + 64 * (size_t)m->tp_rank, dh, 64, ncclUint8, reinterpret_cast<ncclComm_t>(m->nccl), st) !=
      ncclSuccess)
    return -5;
  if (cudaStreamSynchronize(st) != cudaSuccess) return -5;
  std::vector<cudaIpcMemHandle_t> hs(tp);
  cudaMemcpy(hs.data(), dh, 64 * (size_t)tp, cudaMemcpyDeviceToHost);
  cudaFree(dh);
  unsigned long long* flags_host[kMaxFusedTp];
  for (int p = 0; p < tp; ++p) {
    char* pb = base;
    if (p != m->tp_rank) {
      void* q = nullptr;
      if (cudaIpcOpenMemHandle(&q, hs[p], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return -6;
      m->tp_ipc_opened.push_back(q);
      pb = static_cast<char*>(q);
    }
    m->tp_peer_recv[p] = reinterpret_cast<float*>(pb);
    m->tp_peer_hn[p] = reinterpret_cast<bf16*>(pb + part_bytes);
    flags_host[p] = reinterpret_cast<unsigned long long*>(pb + out_bytes);
  }
  m->tp_recv = reinterpret_cast<float*>(base);
  m->tp_hn = reinterpret_cast<bf16*>(base + part_bytes);
  m->tp_flags = reinterpret_cast<unsigned long long*>(base + out_bytes);
  if (cudaMalloc(&m->tp_peer_flags_dev, sizeof(flags_host)) != cudaSuccess) return -3;
  m->allocs.push_back(m->tp_peer_flags_dev);
  cudaMemcpy(m->tp_peer_flags_dev, flags_host, sizeof(flags_host), cudaMemcpyHostToDevice);
  m->tp_fused_rows = max_rows;
  // barrier: every rank has mapped every peer before anyone may write into a peer
  char* one = nullptr;
  if (cudaMalloc(&one, 8) != cudaSuccess) return -3;
  const bool ok = nccl().AllReduce(one, one, 1, ncclUint64, ncclSum, reinterpret_cast<ncclComm_t>(m->nccl), st) ==
                  ncclSuccess;
  cudaStreamSynchronize(st);
  cudaFree(one);
  if (!ok) return -5;
  // NVLS variant on request; any failure leaves the push path in place (collective decision)
  static const bool want_nvls = getenv("SPECEDGE_TP_F4") && std::string(getenv("SPECEDGE_TP_F4")) == "nvls";
  if (want_nvls) {
    const int r = tp_nvls_enable(m, max_rows, st);
    if (r != 0 && getenv("SPECEDGE_DEBUG")) fprintf(stderr, "libspecedge: NVLS setup failed (%d), push path kept\n", r);
  }
  return 0;
}

// ---------------------------------------------------------------------------------------------
// NEXT-F4, NVLS variant (SPECEDGE_TP_F4=nvls).  One CUDA multicast object spans the ranks; every
// rank binds its own physical [2][R_max][d] fp32 buffer to it and maps both the buffer (unicast:
// its row-parallel GEMM stores its partial there) and the multicast object (its RMSNorm loads the
// rank sum of its own rows with multimem.ld_reduce: the reduction happens in the NVSwitch, each
// partial crosses NVLink once).  Rank 0 creates the object and exports a POSIX file descriptor; the
// others duplicate it with pidfd_getfd (pid and fd travel through the NCCL communicator).  Buffer
// halves alternate per collective exactly like the push variant's receive buffers.
// ---------------------------------------------------------------------------------------------
namespace {
struct CuDrv {
  bool tried = false, ok = false;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
};
CuDrv& drv() {
  static CuDrv d;
  if (d.tried) return d;
  d.tried = true;
  auto get = [](const char* name) -> void* {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      return nullptr;
    return p;
  };
#define SE_DRV(f) d.f = reinterpret_cast<decltype(d.f)>(get("cu" #f))
  SE_DRV(MulticastCreate);
  SE_DRV(MulticastGetGranularity);
  SE_DRV(MulticastAddDevice);
  SE_DRV(MulticastBindMem);
  SE_DRV(MulticastUnbind);
  SE_DRV(MemCreate);
  SE_DRV(MemRelease);
  SE_DRV(MemAddressReserve);
  SE_DRV(MemAddressFree);
  SE_DRV(MemMap);
  SE_DRV(MemUnmap);
  SE_DRV(MemSetAccess);
  SE_DRV(MemExportToShareableHandle);
  SE_DRV(MemImportFromShareableHandle);
  SE_DRV(DeviceGet);
#undef SE_DRV
  d.ok = d.MulticastCreate && d.MulticastGetGranularity && d.MulticastAddDevice && d.MulticastBindMem &&
         d.MulticastUnbind && d.MemCreate && d.MemRelease && d.MemAddressReserve && d.MemAddressFree && d.MemMap &&
         d.MemUnmap && d.MemSetAccess && d.MemExportToShareableHandle && d.MemImportFromShareableHandle && d.DeviceGet;
  return d;
}
}  // namespace

// Collective (every rank): returns 0, or < 0 with nothing mapped (the caller keeps the push path)
int tp_nvls_enable(specedge_model* m, int max_rows, cudaStream_t st) {
  static const bool dbg = getenv("SPECEDGE_DEBUG") != nullptr;
#define NVLS_STEP(msg) do { if (dbg) { fprintf(stderr, "[nvls rank %d] %s\n", m->tp_rank, msg); fflush(stderr); } } while (0)
  CuDrv& D = drv();
  NVLS_STEP(D.ok ? "driver entry points ok" : "driver entry points missing");
  if (!D.ok || !m->nccl) return -1;
  const int tp = m->tp_size;
  CUdevice dev;
  if (D.DeviceGet(&dev, m->device) != CUDA_SUCCESS) return -1;
  const size_t half = (size_t)max_rows * m->cfg.d;
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)tp;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = 2 * half * sizeof(float);
  if (D.MulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !gran) return -1;
  const size_t bytes = (mp.size + gran - 1) / gran * gran;
  mp.size = bytes;
  // rank 0 creates and exports; (pid, fd) of rank 0 reach every rank through the communicator
  CUmemGenericAllocationHandle mc = 0;
  long long info[2] = {0, -1};   // ranks != 0 contribute (0, -1) to the sum
  int rc = 0;
  int fd0 = -1;
  if (m->tp_rank == 0) {
    int& fd = fd0;
    if (D.MulticastCreate(&mc, &mp) != CUDA_SUCCESS) rc = -2;
    else if (D.MemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS) rc = -2;
    info[0] = (long long)getpid();
    info[1] = rc == 0 ? fd : -1;
  }
  long long* dinfo = nullptr;
  if (cudaMalloc(&dinfo, sizeof(info)) != cudaSuccess) return -3;
  cudaMemcpy(dinfo, info, sizeof(info), cudaMemcpyHostToDevice);
  NVLS_STEP("created / exported; exchanging (pid, fd)");
  const bool bc = nccl().AllReduce(dinfo, dinfo, 2, ncclInt64, ncclSum, reinterpret_cast<ncclComm_t>(m->nccl), st) ==
                  ncclSuccess;   // ranks != 0 contribute zeros
  cudaStreamSynchronize(st);
  cudaMemcpy(info, dinfo, sizeof(info), cudaMemcpyDeviceToHost);
  cudaFree(dinfo);
  info[1] += (tp - 1);   // the tp - 1 other ranks each contributed -1
  if (!bc || info[1] < 0) return -4;
  if (m->tp_rank != 0) {
    const int pidfd = (int)syscall(SYS_pidfd_open, (pid_t)info[0], 0);
    const int fd = pidfd >= 0 ? (int)syscall(SYS_pidfd_getfd, pidfd, (int)info[1], 0) : -1;
    if (pidfd >= 0) close(pidfd);
    if (fd < 0 || D.MemImportFromShareableHandle(&mc, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) !=
                      CUDA_SUCCESS)
      rc = -5;
    if (fd >= 0) close(fd);
  }
  NVLS_STEP(rc == 0 ? "imported" : "import failed");
  if (rc == 0 && D.MulticastAddDevice(mc, dev) != CUDA_SUCCESS) rc = -6;
  NVLS_STEP(rc == 0 ? "device added" : "add device failed");
  // every rank must have added its device before memory is bound: barrier, and agree on success
  int* dok = nullptr;
  if (cudaMalloc(&dok, sizeof(int)) != cudaSuccess) return -3;
  const int fail = rc != 0 ? 1 : 0;
  cudaMemcpy(dok, &fail, sizeof(int), cudaMemcpyHostToDevice);
  nccl().AllReduce(dok, dok, 1, ncclInt32, ncclSum, reinterpret_cast<ncclComm_t>(m->nccl), st);
  cudaStreamSynchronize(st);
  int nfail = 1;
  cudaMemcpy(&nfail, dok, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(dok);
  if (fd0 >= 0) close(fd0);   // every rank holds its own reference now
  if (nfail) return -7;
  // this rank's physical memory, bound into the object and mapped twice
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = m->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;   // as the multicast object's
  CUmemGenericAllocationHandle mem = 0;
  CUdeviceptr uva = 0, mva = 0;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = m->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUresult cr = D.MemCreate(&mem, bytes, &ap, 0);
  bool ok = cr == CUDA_SUCCESS;
  if (dbg) fprintf(stderr, "[nvls rank %d] cuMemCreate(%zu) -> %d\n", m->tp_rank, bytes, (int)cr);
  bool bound = false;
  if (ok) {
    cr = D.MulticastBindMem(mc, 0, mem, 0, bytes, 0);
    bound = ok = cr == CUDA_SUCCESS;
    if (dbg) fprintf(stderr, "[nvls rank %d] cuMulticastBindMem -> %d (gran %zu)\n", m->tp_rank, (int)cr, gran);
  }
  ok = ok && D.MemAddressReserve(&uva, bytes, gran, 0, 0) == CUDA_SUCCESS;
  ok = ok && D.MemMap(uva, bytes, 0, mem, 0) == CUDA_SUCCESS;
  ok = ok && D.MemSetAccess(uva, bytes, &acc, 1) == CUDA_SUCCESS;
  ok = ok && D.MemAddressReserve(&mva, bytes, gran, 0, 0) == CUDA_SUCCESS;
  ok = ok && D.MemMap(mva, bytes, 0, mc, 0) == CUDA_SUCCESS;
  ok = ok && D.MemSetAccess(mva, bytes, &acc, 1) == CUDA_SUCCESS;
  // agree again (a rank that failed here leaves the others on the push path as well)
  int* dok2 = nullptr;
  cudaMalloc(&dok2, sizeof(int));
  const int fail2 = ok ? 0 : 1;
  cudaMemcpy(dok2, &fail2, sizeof(int), cudaMemcpyHostToDevice);
  nccl().AllReduce(dok2, dok2, 1, ncclInt32, ncclSum, reinterpret_cast<ncclComm_t>(m->nccl), st);
  cudaStreamSynchronize(st);
  cudaMemcpy(&nfail, dok2, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(dok2);
  m->tp_nvls_mem = mem;
  m->tp_nvls_mch = mc;
  m->tp_nvls_uc = reinterpret_cast<float*>(uva);
  m->tp_nvls_mc = reinterpret_cast<float*>(mva);
  m->tp_nvls_bytes = bytes;
  m->tp_nvls_buf = half;
  m->tp_nvls_bound = bound;
  if (nfail) {
    tp_nvls_close(m);
    return -8;
  }
  cudaMemset(m->tp_nvls_uc, 0, bytes);
  cudaDeviceSynchronize();
  m->tp_nvls = true;
  NVLS_STEP("mapped: NVLS on");
#undef NVLS_STEP
  return 0;
}

void tp_nvls_close(specedge_model* m) {
  CuDrv& D = drv();
  if (!D.ok) return;
  cudaDeviceSynchronize();
  const size_t bytes = m->tp_nvls_bytes;
  if (m->tp_nvls_mc) D.MemUnmap(reinterpret_cast<CUdeviceptr>(m->tp_nvls_mc), bytes);
  if (m->tp_nvls_uc) D.MemUnmap(reinterpret_cast<CUdeviceptr>(m->tp_nvls_uc), bytes);
  if (m->tp_nvls_mc) D.MemAddressFree(reinterpret_cast<CUdeviceptr>(m->tp_nvls_mc), bytes);
  if (m->tp_nvls_uc) D.MemAddressFree(reinterpret_cast<CUdeviceptr>(m->tp_nvls_uc), bytes);
  CUdevice dev;
  if (m->tp_nvls_bound && D.DeviceGet(&dev, m->device) == CUDA_SUCCESS) D.MulticastUnbind(m->tp_nvls_mch, dev, 0, bytes);
  m->tp_nvls_bound = false;
  if (m->tp_nvls_mem) D.MemRelease(m->tp_nvls_mem);
  if (m->tp_nvls_mch) D.MemRelease(m->tp_nvls_mch);
  m->tp_nvls_mc = m->tp_nvls_uc = nullptr;
  m->tp_nvls_mem = m->tp_nvls_mch = 0;
  m->tp_nvls = false;
}

void tp_fused_close(specedge_model* m) {
  if (m->tp_nvls_bytes) tp_nvls_close(m);
  for (void* q : m->tp_ipc_opened) cudaIpcCloseMemHandle(q);
  m->tp_ipc_opened.clear();
}

}  // namespace se
