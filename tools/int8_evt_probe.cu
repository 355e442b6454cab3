// int8_evt_probe.cu -- probe (not part of the library): CUTLASS sm100 INT8 GEMM
// with an EVT epilogue D = (acc mod m_batch) stored as uint8 (per-batch
// modulus from a Sm90ScalarBroadcast with a batch stride). Checks exactness
// and times it against the int32-output GEMM.
#include <cstdio>
#include <vector>
#include "cutlass/cutlass.h"
#include "cute/tensor.hpp"
#include "cutlass/gemm/dispatch_policy.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/epilogue/fusion/sm90_callbacks_tma_warpspecialized.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"
using namespace cute;

template <class T> struct ModNonneg;
template <int N>
struct ModNonneg<cutlass::Array<int32_t, N>> {
  CUTLASS_HOST_DEVICE cutlass::Array<int32_t, N> operator()(cutlass::Array<int32_t, N> const &a,
                                                           cutlass::Array<int32_t, N> const &m) const {
    cutlass::Array<int32_t, N> r;
    CUTLASS_PRAGMA_UNROLL
    for (int i = 0; i < N; ++i) {
      const int32_t x = a[i] % m[i];
      r[i] = x < 0 ? x + m[i] : x;
    }
    return r;
  }
};

using TileShape = Shape<_256, _256, _128>;
using ClusterShape = Shape<_2, _1, _1>;
namespace fu = cutlass::epilogue::fusion;
using EVT = fu::Sm90EVT<fu::Sm90Compute<ModNonneg, uint8_t, int32_t, cutlass::FloatRoundStyle::round_to_nearest>,
                        fu::Sm90AccFetch, fu::Sm90ScalarBroadcast<int32_t, Stride<_0, _0, int64_t>>>;
using Epi = typename cutlass::epilogue::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, TileShape, ClusterShape,
    cutlass::epilogue::collective::EpilogueTileAuto, int32_t, int32_t, void, cutlass::layout::RowMajor, 16,
    uint8_t, cutlass::layout::RowMajor, 16, cutlass::epilogue::collective::EpilogueScheduleAuto, EVT>::CollectiveOp;
using Main = typename cutlass::gemm::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, int8_t, cutlass::layout::RowMajor, 16, int8_t,
    cutlass::layout::ColumnMajor, 16, int32_t, TileShape, ClusterShape,
    cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename Epi::SharedStorage))>,
    cutlass::gemm::collective::KernelScheduleAuto>::CollectiveOp;
using Kernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Main, Epi, void>;
using Gemm = cutlass::gemm::device::GemmUniversalAdapter<Kernel>;

__global__ void fill8(int8_t *p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t z = (uint32_t)(i * 2654435761u) ^ seed;
    z ^= z >> 13; z *= 0x5bd1e995u; z ^= z >> 15;
    p[i] = (int8_t)((int)(z % 255) - 127);
  }
}

int main() {
  const int M = 8192, N = 8192, K = 8192, L = 3;
  int8_t *A, *B; uint8_t *D; int32_t *mods;
  cudaMalloc(&A, (size_t)M * K * L); cudaMalloc(&B, (size_t)N * K * L); cudaMalloc(&D, (size_t)M * N * L);
  cudaMalloc(&mods, L * 4);
  int hm[3] = {255, 253, 251};
  cudaMemcpy(mods, hm, 12, cudaMemcpyHostToDevice);
  fill8<<<1024, 256>>>(A, (size_t)M * K * L, 1); fill8<<<1024, 256>>>(B, (size_t)N * K * L, 2);
  using SA = typename Gemm::GemmKernel::StrideA; using SB = typename Gemm::GemmKernel::StrideB;
  using SC = typename Gemm::GemmKernel::StrideC; using SD = typename Gemm::GemmKernel::StrideD;
  SA sa = cutlass::make_cute_packed_stride(SA{}, {M, K, L});
  SB sb = cutlass::make_cute_packed_stride(SB{}, {N, K, L});
  SC sc = cutlass::make_cute_packed_stride(SC{}, {M, N, L});
  SD sd = cutlass::make_cute_packed_stride(SD{}, {M, N, L});
  typename EVT::Arguments fargs{{}, {{0}, {mods}, {Stride<_0, _0, int64_t>{_0{}, _0{}, int64_t(1)}}}, {}};
  typename Gemm::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm, {M, N, K, L}, {A, sa, B, sb},
                                {fargs, nullptr, sc, D, sd}};
  Gemm gemm;
  size_t ws = Gemm::get_workspace_size(args); void *wsp = nullptr; if (ws) cudaMalloc(&wsp, ws);
  printf("can_implement %d\n", (int)gemm.can_implement(args));
  if (gemm.initialize(args, wsp) != cutlass::Status::kSuccess) { printf("init failed\n"); return 1; }
  gemm.run(); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; r++) { cudaEventRecord(e0); gemm.run(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; }
  printf("EVT uint8 mod: %.3f ms  %.1f TOPS  err=%s\n", best, 2.0 * M * N * (double)K * L / best / 1e9, cudaGetErrorString(cudaGetLastError()));
  std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K); std::vector<uint8_t> hD((size_t)M * N);
  int bad = 0;
  for (int b = 0; b < L; b++) {
    cudaMemcpy(hA.data(), A + (size_t)b * M * K, hA.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(hB.data(), B + (size_t)b * N * K, hB.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(hD.data(), D + (size_t)b * M * N, hD.size(), cudaMemcpyDeviceToHost);
    for (int t = 0; t < 32; t++) {
      int i = (t * 7919 + b) % M, j = (t * 104729 + 3 * b) % N;
      long long s = 0;
      for (int k = 0; k < K; k++) s += (long long)hA[(size_t)i * K + k] * hB[(size_t)j * K + k];
      long long r = s % hm[b]; if (r < 0) r += hm[b];
      if (r != hD[(size_t)i * N + j]) bad++;
    }
  }
  printf("exactness: %d / %d mismatches\n", bad, 32 * L);
  return 0;
}
