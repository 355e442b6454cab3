// gather.cu -- the all-gather of the sharded H_eff output over peer memory
// (DESIGN.md §9). Every rank maps the other ranks' full
// output buffers and flag arrays (CUDA IPC over NVLink / NVSwitch); the
// Ozaki CRT epilogue of GEMM4 stores each finished output element into the
// local slab AND into the same slab of every peer's buffer (ozaki.cu), so the
// transfer happens tile by tile inside the producing kernel. This file holds
// the two small kernels around it:
//  * gather_barrier: a flag exchange (release / acquire at system scope):
//    rank r writes `epoch` into slot r of every peer's flag array after its
//    stores, then spins until every slot of its own array reached `epoch`.
//    Flags only grow (epoch counter per context), so they never need a reset.
//    A %globaltimer bound turns a missing peer into an error flag instead of
//    a hang; the flag is sticky until the next tci_gather_register (later
//    barriers return at once) and tci_gather_status reports it.
//  * push_rows: the unfused path (DMMA GEMM4 or the generic tree): the local
//    slab is copied to every peer with 16-byte stores over NVLink.
#include <algorithm>
#include <cstdint>

#include "../tci_internal.h"

namespace tci {
namespace {

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void gather_barrier(const PeerTable t, int rank, int nranks, uint32_t epoch, int *err,
                               unsigned long long timeout_ns) {
  const int j = threadIdx.x;
  if (j < nranks) {
    // everything this rank stored before (previous kernels on the stream,
    // local and remote) is ordered before the flag
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release_sys(static_cast<uint32_t *>(t.flags[j]) + rank, epoch);
  }
  __syncthreads();
  // sticky error: once a barrier of this registration timed out, later
  // barriers do not wait again (the run is already reported as failed)
  if (*reinterpret_cast<volatile int *>(err)) return;
  if (j < nranks) {
    const uint32_t *mine = static_cast<const uint32_t *>(t.flags[rank]) + j;
    const uint64_t t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(err, 1);
        break;
      }
      __nanosleep(256);
    }
  }
}

__global__ void push_rows(const int4 *__restrict__ src, const PeerTable t, int rank, int nranks, size_t off16,
                          size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
    const int4 v = __ldg(src + i);
#pragma unroll 1
    for (int j = 0; j < nranks; j++)
      if (j != rank) static_cast<int4 *>(t.full[j])[off16 + i] = v;
  }
}

}  // namespace

// Load both kernels now (CUDA lazy loading would otherwise load them at their
// first launch, which must not happen while a barrier of this device spins)
cudaError_t gather_preload() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, gather_barrier);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, push_rows);
  return e;
}

cudaError_t launch_gather_barrier(const PeerTable &t, int rank, int nranks, uint32_t epoch, int *err,
                                  double timeout_s, cudaStream_t s, int64_t *launches) {
  gather_barrier<<<1, 32, 0, s>>>(t, rank, nranks, epoch, err, (unsigned long long)(timeout_s * 1e9));
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_push_rows(const void *src, const PeerTable &t, int rank, int nranks, size_t offset_bytes,
                             size_t bytes, cudaStream_t s, int64_t *launches) {
  if (nranks <= 1 || bytes == 0) return cudaSuccess;
  if (bytes % 16 || offset_bytes % 16 || (uintptr_t)src % 16) return cudaErrorInvalidValue;
  const size_t n16 = bytes / 16;
  const unsigned blocks = (unsigned)std::min<size_t>((n16 + 255) / 256, 148 * 4);
  push_rows<<<blocks, 256, 0, s>>>(static_cast<const int4 *>(src), t, rank, nranks, offset_bytes / 16, n16);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tci
