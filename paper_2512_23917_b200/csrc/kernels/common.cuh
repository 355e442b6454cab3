// common.cuh -- small PTX helpers shared by the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tci {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero-fill: copies `src_bytes` (0..CP) bytes, zero-fills the rest.
template <int CP>
__device__ __forceinline__ void cp_async_zfill(void *smem, const void *gmem, int src_bytes) {
  static_assert(CP == 4 || CP == 8 || CP == 16, "cp.async size");
  if constexpr (CP == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(src_bytes));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "n"(CP), "r"(src_bytes));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// FP64 tensor-core MMA (DMMA): D[8x8] += A[8x4] (row) * B[4x8] (col).
// Fragment ownership (lane l): A[l/4][l%4], B[l%4][l/4], C[l/4][2*(l%4)+{0,1}].
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

}  // namespace tci
