// int8_probe.cu -- feasibility probe (not part of the library): a CUTLASS 4.5
// sm100 tcgen05 INT8 GEMM (kind::i8, TMA, TMEM accumulators, 2-SM cluster)
// built from the CollectiveBuilder, timed on M=N=K=8192 and on the
// H_eff GEMM4 shape, exactness checked against an int64 host reference on a
// sample. Decides whether the Ozaki-scheme path is viable.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cutlass/cutlass.h"
#include "cute/tensor.hpp"
#include "cutlass/gemm/dispatch_policy.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"

using namespace cute;

using ElementA = int8_t;
using LayoutA = cutlass::layout::RowMajor;      // K-major
using ElementB = int8_t;
using LayoutB = cutlass::layout::ColumnMajor;   // K-major
using ElementC = int32_t;
using LayoutC = cutlass::layout::RowMajor;
using ElementAcc = int32_t;
constexpr int AlignA = 16, AlignB = 16, AlignC = 4;

template <class TileShape, class ClusterShape>
struct GemmT {
  using Epi = typename cutlass::epilogue::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, TileShape, ClusterShape,
      cutlass::epilogue::collective::EpilogueTileAuto, ElementAcc, ElementAcc, ElementC, LayoutC, AlignC,
      ElementC, LayoutC, AlignC, cutlass::epilogue::collective::EpilogueScheduleAuto>::CollectiveOp;
  using Main = typename cutlass::gemm::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, ElementA, LayoutA, AlignA, ElementB, LayoutB, AlignB,
      ElementAcc, TileShape, ClusterShape,
      cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename Epi::SharedStorage))>,
      cutlass::gemm::collective::KernelScheduleAuto>::CollectiveOp;
  using Kernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Main, Epi, void>;
  using Gemm = cutlass::gemm::device::GemmUniversalAdapter<Kernel>;
};

__global__ void fill8(int8_t *p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t z = (uint32_t)(i * 2654435761u) ^ seed;
    z ^= z >> 13; z *= 0x5bd1e995u; z ^= z >> 15;
    p[i] = (int8_t)((int)(z % 255) - 127);
  }
}

template <class G>
double run(int M, int N, int K, int L, bool check) {
  using Gemm = typename G::Gemm;
  using StrideA = typename Gemm::GemmKernel::StrideA;
  using StrideB = typename Gemm::GemmKernel::StrideB;
  using StrideC = typename Gemm::GemmKernel::StrideC;
  using StrideD = typename Gemm::GemmKernel::StrideD;
  int8_t *A, *B;
  int32_t *C;
  cudaMalloc(&A, (size_t)M * K * L);
  cudaMalloc(&B, (size_t)N * K * L);
  cudaMalloc(&C, (size_t)M * N * L * 4);
  fill8<<<1024, 256>>>(A, (size_t)M * K * L, 1);
  fill8<<<1024, 256>>>(B, (size_t)N * K * L, 2);
  StrideA sA = cutlass::make_cute_packed_stride(StrideA{}, {M, K, L});
  StrideB sB = cutlass::make_cute_packed_stride(StrideB{}, {N, K, L});
  StrideC sC = cutlass::make_cute_packed_stride(StrideC{}, {M, N, L});
  StrideD sD = cutlass::make_cute_packed_stride(StrideD{}, {M, N, L});
  typename Gemm::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm, {M, N, K, L}, {A, sA, B, sB},
                                {{1, 0}, C, sC, C, sD}};
  Gemm gemm;
  size_t ws = Gemm::get_workspace_size(args);
  void *wsp = nullptr;
  if (ws) cudaMalloc(&wsp, ws);
  if (gemm.can_implement(args) != cutlass::Status::kSuccess) { printf("cannot implement\n"); return -1; }
  if (gemm.initialize(args, wsp) != cutlass::Status::kSuccess) { printf("init failed\n"); return -1; }
  gemm.run();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(e0);
    gemm.run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  if (err) printf("cuda error %s\n", cudaGetErrorString(err));
  if (check) {
    std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K);
    std::vector<int32_t> hC((size_t)M * N);
    cudaMemcpy(hA.data(), A, hA.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(hB.data(), B, hB.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int t = 0; t < 64; t++) {
      int i = (t * 7919) % M, j = (t * 104729) % N;
      long long s = 0;
      for (int k = 0; k < K; k++) s += (long long)hA[(size_t)i * K + k] * hB[(size_t)j * K + k];
      if (s != hC[(size_t)i * N + j]) bad++;
    }
    printf("  exactness check: %d / 64 mismatches\n", bad);
  }
  cudaFree(A); cudaFree(B); cudaFree(C);
  if (wsp) cudaFree(wsp);
  return best / 1e3;
}

int main() {
  using G2 = GemmT<Shape<_256, _256, _128>, Shape<_2, _1, _1>>;
  using G1 = GemmT<Shape<_128, _256, _128>, Shape<_1, _1, _1>>;
  struct { int M, N, K, L; } shapes[] = {{8192, 8192, 8192, 1}, {16384, 8192, 40960, 1}, {20480, 32768, 8192, 1}};
  for (auto s : shapes) {
    double t2 = run<G2>(s.M, s.N, s.K, s.L, s.M == 8192);
    double t1 = run<G1>(s.M, s.N, s.K, s.L, false);
    const double ops = 2.0 * s.M * s.N * (double)s.K * s.L;
    printf("M=%d N=%d K=%d: 2SM 256x256x128 %.3f ms %.1f TOPS | 1SM 128x256x128 %.3f ms %.1f TOPS\n", s.M, s.N,
           s.K, t2 * 1e3, ops / t2 / 1e12, t1 * 1e3, ops / t1 / 1e12);
  }
  return 0;
}
