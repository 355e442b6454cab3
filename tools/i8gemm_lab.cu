// i8gemm_lab.cu -- standalone check + timing of the hand-written tcgen05
// INT8 residue GEMM (paper_2512_23917_b200/csrc/kernels/i8gemm.cu):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/i8gemm_lab.cu -o tools/i8gemm_lab && tools/i8gemm_lab
// Every output of small ragged problems and 4096 sampled outputs of the
// bench-sized ones are compared with a plain int64 dot product mod m.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2512_23917_b200/csrc/kernels/i8gemm.cu"
#include "../paper_2512_23917_b200/csrc/launch_cache.cpp"

#ifdef WITH_CUTLASS
// the library INT8 GEMM the round-1 build used, for an A/B in the same process
#include "cutlass/cutlass.h"
#include "cute/tensor.hpp"
#include "cutlass/gemm/dispatch_policy.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/epilogue/fusion/sm90_callbacks_tma_warpspecialized.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"
namespace cl {
using namespace cute;
template <class T> struct ModNonneg;
template <int N> struct ModNonneg<cutlass::Array<int32_t, N>> {
  CUTLASS_HOST_DEVICE cutlass::Array<int32_t, N> operator()(cutlass::Array<int32_t, N> const &a,
                                                           cutlass::Array<int32_t, N> const &m) const {
    cutlass::Array<int32_t, N> r;
    for (int i = 0; i < N; ++i) { const int32_t x = a[i] % m[i]; r[i] = x < 0 ? x + m[i] : x; }
    return r;
  }
};
namespace fu = cutlass::epilogue::fusion;
using ModEVT = fu::Sm90EVT<fu::Sm90Compute<ModNonneg, uint8_t, int32_t, cutlass::FloatRoundStyle::round_to_nearest>,
                           fu::Sm90AccFetch, fu::Sm90ScalarBroadcast<int32_t, Stride<_0, _0, int64_t>>>;
using TileShape = Shape<_256, _256, _128>;
using ClusterShape = Shape<_2, _1, _1>;
using Epi = typename cutlass::epilogue::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, TileShape, ClusterShape,
    cutlass::epilogue::collective::EpilogueTileAuto, int32_t, int32_t, void, cutlass::layout::RowMajor, 16,
    uint8_t, cutlass::layout::RowMajor, 16, cutlass::epilogue::collective::EpilogueScheduleAuto, ModEVT>::CollectiveOp;
using Main = typename cutlass::gemm::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, int8_t, cutlass::layout::RowMajor, 16, int8_t,
    cutlass::layout::ColumnMajor, 16, int32_t, TileShape, ClusterShape,
    cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename Epi::SharedStorage))>,
    cutlass::gemm::collective::KernelScheduleAuto>::CollectiveOp;
using I8Kernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Main, Epi, void>;
using I8Gemm = cutlass::gemm::device::GemmUniversalAdapter<I8Kernel>;
static void *cws = nullptr;
cudaError_t run(const int8_t *A, const int8_t *B, uint8_t *D, int32_t *bmod, int M, int N, int K, int L) {
  using SA = typename I8Gemm::GemmKernel::StrideA; using SB = typename I8Gemm::GemmKernel::StrideB;
  using SC = typename I8Gemm::GemmKernel::StrideC; using SD = typename I8Gemm::GemmKernel::StrideD;
  SA sa = cutlass::make_cute_packed_stride(SA{}, {M, K, L}); SB sb = cutlass::make_cute_packed_stride(SB{}, {N, K, L});
  SC sc = cutlass::make_cute_packed_stride(SC{}, {M, N, L}); SD sd = cutlass::make_cute_packed_stride(SD{}, {M, N, L});
  typename ModEVT::Arguments fargs{{}, {{0}, {bmod}, {Stride<_0, _0, int64_t>{_0{}, _0{}, int64_t(1)}}}, {}};
  typename I8Gemm::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm, {M, N, K, L},
                                  {A, sa, B, sb}, {fargs, nullptr, sc, D, sd}};
  args.scheduler.max_swizzle_size = 8;
  args.scheduler.raster_order = cutlass::gemm::kernel::detail::RasterOrderOptions::AlongM;
  I8Gemm g;
  if (g.can_implement(args) != cutlass::Status::kSuccess) return cudaErrorNotSupported;
  if (!cws) cudaMalloc(&cws, 64 << 20);
  if (g.initialize(args, cws, 0) != cutlass::Status::kSuccess) return cudaErrorUnknown;
  return g.run(0) == cutlass::Status::kSuccess ? cudaSuccess : cudaErrorUnknown;
}
}  // namespace cl
#endif

using namespace tci;
using namespace tci::i8g;

__global__ void fill_rand(int8_t *p, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = (int8_t)((int)(z % 255) - 127);
  }
}

// reference: sampled (b, m, n) or all when idx == nullptr
__global__ void ref_kernel(const int8_t *A, const int8_t *B, int64_t M, int64_t N, int64_t Kp, int L, int per_mod,
                           const int64_t *idx, int64_t nidx, const int *mods, uint8_t *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nidx) return;
  const int64_t e = idx ? idx[i] : i;
  const int64_t b = e / (M * N), m = (e / N) % M, n = e % N;
  long long acc = 0;
  for (int64_t k = 0; k < Kp; k++) acc += (int)A[(b * M + m) * Kp + k] * (int)B[(b * N + n) * Kp + k];
  const int md = mods[b / per_mod];
  long long r = acc % md;
  if (r < 0) r += md;
  out[i] = (uint8_t)r;
}

static const int hm[16] = {255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193, 1};

static int check(int64_t M, int64_t N, int64_t Kp, int L, int per_mod, bool full, int reps) {
  int8_t *A, *B;
  uint8_t *D, *R;
  int64_t *idx = nullptr;
  int *mods;
  cudaMalloc(&A, (size_t)L * M * Kp);
  cudaMalloc(&B, (size_t)L * N * Kp);
  cudaMalloc(&D, (size_t)L * M * N);
  cudaMalloc(&mods, sizeof hm);
  int *ctr;
  cudaMalloc(&ctr, 4);
  cudaMemcpy(mods, hm, sizeof hm, cudaMemcpyHostToDevice);
  fill_rand<<<1024, 256>>>(A, (size_t)L * M * Kp, 1);
  fill_rand<<<1024, 256>>>(B, (size_t)L * N * Kp, 2);
  cudaMemset(D, 0xAB, (size_t)L * M * N);
  int64_t nidx = full ? L * M * N : 4096;
  std::vector<int64_t> hidx;
  if (!full) {
    srand(7);
    for (int64_t i = 0; i < nidx; i++) {
      int64_t b = rand() % L, m = (i < 64) ? (i % 2 ? M - 1 : 0) : rand() % M, n = (i % 3 == 0) ? N - 1 : rand() % N;
      hidx.push_back((b * M + m) * N + n);
    }
    cudaMalloc(&idx, nidx * 8);
    cudaMemcpy(idx, hidx.data(), nidx * 8, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&R, nidx);
  cudaError_t e = launch_i8gemm(A, B, D, M, N, Kp, L, per_mod, hm, (L + per_mod - 1) / per_mod, ctr, 0, nullptr);
  if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("run: %s\n", cudaGetErrorString(e)); return 1; }
  ref_kernel<<<(unsigned)((nidx + 127) / 128), 128>>>(A, B, M, N, Kp, L, per_mod, idx, nidx, mods, R);
  cudaDeviceSynchronize();
  std::vector<uint8_t> hr(nidx), hd((size_t)L * M * N);
  cudaMemcpy(hr.data(), R, nidx, cudaMemcpyDeviceToHost);
  cudaMemcpy(hd.data(), D, hd.size(), cudaMemcpyDeviceToHost);
  int64_t bad = 0;
  for (int64_t i = 0; i < nidx; i++) {
    const int64_t eidx = full ? i : hidx[i];
    if (hd[eidx] != hr[i]) {
      if (bad < 5) printf("  mismatch at %lld: got %d want %d\n", (long long)eidx, hd[eidx], hr[i]);
      bad++;
    }
  }
  double ms = 0;
  if (reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch_i8gemm(A, B, D, M, N, Kp, L, per_mod, hm, (L + per_mod - 1) / per_mod, ctr, 0, nullptr);
    cudaEventRecord(a);
    for (int r = 0; r < reps; r++) launch_i8gemm(A, B, D, M, N, Kp, L, per_mod, hm, (L + per_mod - 1) / per_mod, ctr, 0, nullptr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    ms = t / reps;
  }
  double ms_cl = 0;
#ifdef WITH_CUTLASS
  if (reps) {
    int32_t *bm;
    std::vector<int32_t> hb(L);
    for (int b = 0; b < L; b++) hb[b] = hm[b / per_mod];
    cudaMalloc(&bm, L * 4);
    cudaMemcpy(bm, hb.data(), L * 4, cudaMemcpyHostToDevice);
    cl::run(A, B, D, bm, (int)M, (int)N, (int)Kp, L);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; r++) cl::run(A, B, D, bm, (int)M, (int)N, (int)Kp, L);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    ms_cl = t / reps;
    cudaFree(bm);
  }
#endif
  const double ops = 2.0 * M * N * Kp * L;
  printf("M=%lld N=%lld K=%lld L=%d: %lld/%lld mismatches%s", (long long)M, (long long)N, (long long)Kp, L,
         (long long)bad, (long long)nidx, full ? " (all)" : " (sampled)");
  if (reps) printf("  %.3f ms  %.1f TOPS", ms, ops / ms * 1e-9);
  if (ms_cl > 0) printf("  | CUTLASS %.3f ms  %.1f TOPS", ms_cl, ops / ms_cl * 1e-9);
  printf("\n");
  cudaFree(A); cudaFree(B); cudaFree(D); cudaFree(R); cudaFree(mods); cudaFree(ctr);
  if (idx) cudaFree(idx);
  return bad != 0;
}

int main(int argc, char **argv) {
  int fails = 0;
  if (argc > 1 && !strcmp(argv[1], "kscan")) {   // per-tile overhead: fixed M x N (GEMM1 chunk), K varied
    const int ks[] = {1024, 2048, 4096, 8192, 16384};
    for (int k : ks) fails += check(9216, 16384, k, 30, 2, false, 3);
    fails += check(10752, 4096, 20480, 30, 2, false, 3);   // GEMM4 chunk
    printf(fails ? "FAIL\n" : "ALL OK\n");
    return fails;
  }
  if (argc > 1 && !strcmp(argv[1], "sweep")) {   // L2-policy sweep on the bench chunk shapes
    const int mbs[] = {24, 32, 48, 64, 96, 1000};
    for (int mb : mbs) {
      g_i8_res_mb = mb;
      printf("resident budget %d MB\n", mb);
      fails += check(9216, 16384, 4096, 42, 3, false, 3);
      fails += check(7680, 4096, 20480, 42, 3, false, 3);
    }
    printf(fails ? "FAIL\n" : "ALL OK\n");
    return fails;
  }
  fails += check(256, 256, 128, 1, 1, true, 0);
  fails += check(300, 272, 192, 3, 3, true, 0);
  fails += check(513, 528, 1088, 4, 1, true, 0);
  fails += check(1024, 1024, 4096, 6, 3, false, 3);
  if (argc > 1) {
    fails += check(9216, 16384, 4096, 42, 3, false, 3);    // bench GEMM1 chunk
    fails += check(7680, 4096, 20480, 42, 3, false, 3);    // bench GEMM4 chunk
  }
  printf(fails ? "FAIL\n" : "ALL OK\n");
  return fails;
}
