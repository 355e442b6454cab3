// gemm_f32.cu -- fp32 / complex64 GEMM over fused legs (SURVEY 8(a4) fp32
// path). 1xTF32 / bf16 tensor-core variants cannot meet the 1e-5 relative-
// Frobenius parity bar on random data (R20), and neither can fp32
// accumulation once a long sum cancels (measured: 5.8e-5 for a K = 8880 full
// contraction). So products of the fp32 inputs are formed and summed in
// fp64 (the products are exact in fp64) and each result is rounded to fp32
// once: error <= one fp32 rounding plus the fp64 sum error.
//
// CTA tile 128x128 (real) / 64x64 (complex), BK = 8, 256 threads, each thread
// an 8x8 (real) or 4x4 (complex) register tile; register-prefetched double
// buffer. Operand strides are generic: the loader maps consecutive threads to
// whichever of the two legs has unit stride, so global reads coalesce for any
// of the four operand layouts.
#include <cstdlib>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

template <typename E>
struct Ops;
template <>
struct Ops<float> {
  using Acc = double;
  static __device__ __forceinline__ float zero() { return 0.f; }
  static __device__ __forceinline__ Acc azero() { return 0.0; }
  static __device__ __forceinline__ Acc wide(float a) { return (double)a; }
  static __device__ __forceinline__ void mac(Acc &c, Acc a, Acc b) { c = fma(a, b, c); }
  static __device__ __forceinline__ float out(Acc c) { return (float)c; }
};
template <>
struct Ops<float2> {
  using Acc = double2;
  static __device__ __forceinline__ float2 zero() { return make_float2(0.f, 0.f); }
  static __device__ __forceinline__ Acc azero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ Acc wide(float2 a) { return make_double2(a.x, a.y); }
  static __device__ __forceinline__ void mac(Acc &c, Acc a, Acc b) {
    const double ax = a.x, ay = a.y, bx = b.x, by = b.y;
    c.x = fma(ax, bx, c.x);
    c.x = fma(-ay, by, c.x);
    c.y = fma(ax, by, c.y);
    c.y = fma(ay, bx, c.y);
  }
  static __device__ __forceinline__ float2 out(Acc c) { return make_float2((float)c.x, (float)c.y); }
};

template <typename E, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const GemmProblem p, int tiles_m, int tiles_n) {
  static_assert((BM / TM) * (BN / TN) == 256, "256 threads");
  using Acc = typename Ops<E>::Acc;
  // operands are widened to fp64 once, when staged (products exact, R20)
  __shared__ Acc As[2][BK][BM];
  __shared__ Acc Bs[2][BK][BN];
  // the Ozaki guard's gated recomputation (R34): nothing to do unless *run_if
  if (p.run_if && *reinterpret_cast<const volatile int *>(p.run_if) == 0) return;
  const int tid = threadIdx.x;
  const int tile_m = blockIdx.x / tiles_n, tile_n = blockIdx.x % tiles_n;
  const int64_t m0 = (int64_t)tile_m * BM, n0 = (int64_t)tile_n * BN;
  const E *A = static_cast<const E *>(p.A);
  const E *B = static_cast<const E *>(p.B);
  E *C = static_cast<E *>(p.C);
  int64_t Kl = p.K;
  typename Ops<E>::Acc *Pz = nullptr;   // split-K partial (fp64 accumulators)
  if (p.splitk > 1) {
    const int64_t kb = (int64_t)blockIdx.z * p.k_chunk;
    Kl = p.K - kb < p.k_chunk ? p.K - kb : p.k_chunk;
    A += kb * p.a_sk;
    B += kb * p.b_sk;
    Pz = static_cast<typename Ops<E>::Acc *>(p.partial) + (int64_t)blockIdx.z * p.M * p.N;
  }
  const bool a_mfast = (p.a_sk != 1);   // canonical: a_sk == 1 or a_sm == 1
  const bool b_nfast = (p.b_sk != 1);
  constexpr int LA = BM * BK / 256, LB = BN * BK / 256;
  E ra[LA], rb[LB];

  auto gload = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < LA; i++) {
      const int idx = tid + i * 256;
      int m, k;
      if (a_mfast) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      const int64_t gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < p.M && gk < Kl) ? A[gm * p.a_sm + gk * p.a_sk] : Ops<E>::zero();
    }
#pragma unroll
    for (int i = 0; i < LB; i++) {
      const int idx = tid + i * 256;
      int n, k;
      if (b_nfast) { k = idx / BN; n = idx % BN; } else { n = idx / BK; k = idx % BK; }
      const int64_t gn = n0 + n, gk = k0 + k;
      rb[i] = (gn < p.N && gk < Kl) ? B[gk * p.b_sk + gn * p.b_sn] : Ops<E>::zero();
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; i++) {
      const int idx = tid + i * 256;
      int m, k;
      if (a_mfast) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      As[buf][k][m] = Ops<E>::wide(ra[i]);
    }
#pragma unroll
    for (int i = 0; i < LB; i++) {
      const int idx = tid + i * 256;
      int n, k;
      if (b_nfast) { k = idx / BN; n = idx % BN; } else { n = idx / BK; k = idx % BK; }
      Bs[buf][k][n] = Ops<E>::wide(rb[i]);
    }
  };

  const int ty = tid / (BN / TN), tx = tid % (BN / TN);
  typename Ops<E>::Acc acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) acc[i][j] = Ops<E>::azero();

  const int KT = (int)((Kl + BK - 1) / BK);
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < KT; kt++) {
    const int buf = kt & 1;
    if (kt + 1 < KT) gload((int64_t)(kt + 1) * BK);
#pragma unroll
    for (int k = 0; k < BK; k++) {
      Acc a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; i++) a[i] = As[buf][k][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; j++) b[j] = Bs[buf][k][tx + j * (BN / TN)];   // conflict-free
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) Ops<E>::mac(acc[i][j], a[i], b[j]);
    }
    if (kt + 1 < KT) {
      sstore(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < TM; i++) {
    const int64_t m = m0 + ty * TM + i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int64_t n = n0 + tx + j * (BN / TN);
      if (n >= p.N) continue;
      if (Pz) Pz[m * p.N + n] = acc[i][j];
      else C[p.c_row ? p.c_row[m] + p.c_col[n] : m * p.c_sm + n] = Ops<E>::out(acc[i][j]);
    }
  }
}

// ---------------------------------------------------------------------------
// float32 on the FP64 tensor cores (DMMA m8n8k4): the operands are widened to
// fp64 exactly while they are staged (as the SIMT kernel above), then each warp
// runs DMMAs on fragments read from shared memory instead of one DFMA per
// product -- 256 products per warp instruction, ~1/20 of the SIMT kernel's
// shared-memory traffic per product, so the FP64 datapath (shared by DFMA and
// DMMA) is kept busy. Same R20 arithmetic: exact products, fp64 sums in a
// fixed k order (ascending, 4 per DMMA), one rounding to fp32.
// CTA BM x BN (128 x 128: 16 warps; 128 x 64 / 64 x 128 for narrow outputs:
// 8 warps), warp tiles 32 x 32 (4 x 4 accumulator fragments), BK 16 with a
// register-prefetched double buffer; rows of the staged tiles padded by 8
// doubles (fragment reads hit each bank pair at most twice: the 2-wavefront
// minimum of a 256-byte read).
// ---------------------------------------------------------------------------
constexpr int kFdBK = 16, kFdPad = 8;
template <int BM, int BN>
constexpr size_t fd_smem() { return (size_t)2 * kFdBK * ((BM + kFdPad) + (BN + kFdPad)) * sizeof(double); }

template <int BM, int BN>
__global__ void __launch_bounds__((BM / 32) * (BN / 32) * 32)
    gemm_f32_dmma_kernel(const GemmProblem p, int tiles_m, int tiles_n) {
  constexpr int BK = kFdBK, LDA = BM + kFdPad, LDB = BN + kFdPad;
  constexpr int WX = BN / 32, NT = (BM / 32) * WX * 32;
  extern __shared__ __align__(16) double fd_sm[];
  double (*As)[BK][LDA] = reinterpret_cast<double (*)[BK][LDA]>(fd_sm);
  double (*Bs)[BK][LDB] = reinterpret_cast<double (*)[BK][LDB]>(fd_sm + 2 * BK * LDA);
  if (p.run_if && *reinterpret_cast<const volatile int *>(p.run_if) == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile_m = blockIdx.x / tiles_n, tile_n = blockIdx.x % tiles_n;
  const int64_t m0 = (int64_t)tile_m * BM, n0 = (int64_t)tile_n * BN;
  const float *A = static_cast<const float *>(p.A);
  const float *B = static_cast<const float *>(p.B);
  float *C = static_cast<float *>(p.C);
  int64_t Kl = p.K;
  double *Pz = nullptr;
  if (p.splitk > 1) {
    const int64_t kb = (int64_t)blockIdx.z * p.k_chunk;
    Kl = p.K - kb < p.k_chunk ? p.K - kb : p.k_chunk;
    A += kb * p.a_sk;
    B += kb * p.b_sk;
    Pz = static_cast<double *>(p.partial) + (int64_t)blockIdx.z * p.M * p.N;
  }
  const bool a_mfast = (p.a_sk != 1), b_nfast = (p.b_sk != 1);
  constexpr int LA = BM * BK / NT, LB = BN * BK / NT;
  float ra[LA], rb[LB];
  auto gload = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < LA; i++) {
      const int idx = tid + i * NT;
      int m, k;
      if (a_mfast) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      const int64_t gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < p.M && gk < Kl) ? A[gm * p.a_sm + gk * p.a_sk] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < LB; i++) {
      const int idx = tid + i * NT;
      int n, k;
      if (b_nfast) { k = idx / BN; n = idx % BN; } else { n = idx / BK; k = idx % BK; }
      const int64_t gn = n0 + n, gk = k0 + k;
      rb[i] = (gn < p.N && gk < Kl) ? B[gk * p.b_sk + gn * p.b_sn] : 0.f;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; i++) {
      const int idx = tid + i * NT;
      int m, k;
      if (a_mfast) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      As[buf][k][m] = (double)ra[i];
    }
#pragma unroll
    for (int i = 0; i < LB; i++) {
      const int idx = tid + i * NT;
      int n, k;
      if (b_nfast) { k = idx / BN; n = idx % BN; } else { n = idx / BK; k = idx % BK; }
      Bs[buf][k][n] = (double)rb[i];
    }
  };
  const int wm = (warp / WX) * 32, wn = (warp % WX) * 32;
  const int fr = lane >> 2, fk = lane & 3;   // fragment row / k of this lane
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (int)((Kl + BK - 1) / BK);
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < KT; kt++) {
    const int buf = kt & 1;
    if (kt + 1 < KT) gload((int64_t)(kt + 1) * BK);
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) a[i] = As[buf][k4 + fk][wm + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 4; j++) b[j] = Bs[buf][k4 + fk][wn + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) dmma884(acc[i][j], a[i], b[j]);
    }
    if (kt + 1 < KT) {
      sstore(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int64_t m = m0 + wm + 8 * i + fr;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t n = n0 + wn + 8 * j + 2 * fk + h;
        if (n >= p.N) continue;
        if (Pz) Pz[m * p.N + n] = acc[i][j][h];
        else C[p.c_row ? p.c_row[m] + p.c_col[n] : m * p.c_sm + n] = (float)acc[i][j][h];
      }
  }
}

// complex64 on the FP64 tensor cores: the same staging (re / im planes widened
// to fp64), 4M with exact products: Cr += Ar Br + (-Ai) Bi, Ci += Ar Bi + Ai Br
// (four DMMAs per fragment pair, fixed order). CTA 64 x 64, 8 warps of 32 x 16.
constexpr int kCdBM = 64, kCdBN = 64;
constexpr size_t cd_smem() { return (size_t)2 * 2 * kFdBK * ((kCdBM + kFdPad) + (kCdBN + kFdPad)) * sizeof(double); }

__global__ void __launch_bounds__(256, 2) gemm_c64_dmma_kernel(const GemmProblem p, int tiles_m, int tiles_n) {
  constexpr int BM = kCdBM, BN = kCdBN, BK = kFdBK, LDA = BM + kFdPad, LDB = BN + kFdPad, NT = 256;
  extern __shared__ __align__(16) double cd_sm[];
  double (*Ar)[BK][LDA] = reinterpret_cast<double (*)[BK][LDA]>(cd_sm);
  double (*Ai)[BK][LDA] = reinterpret_cast<double (*)[BK][LDA]>(cd_sm + 2 * BK * LDA);
  double (*Br)[BK][LDB] = reinterpret_cast<double (*)[BK][LDB]>(cd_sm + 4 * BK * LDA);
  double (*Bi)[BK][LDB] = reinterpret_cast<double (*)[BK][LDB]>(cd_sm + 4 * BK * LDA + 2 * BK * LDB);
  if (p.run_if && *reinterpret_cast<const volatile int *>(p.run_if) == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile_m = blockIdx.x / tiles_n, tile_n = blockIdx.x % tiles_n;
  const int64_t m0 = (int64_t)tile_m * BM, n0 = (int64_t)tile_n * BN;
  const float2 *A = static_cast<const float2 *>(p.A);
  const float2 *B = static_cast<const float2 *>(p.B);
  float2 *C = static_cast<float2 *>(p.C);
  int64_t Kl = p.K;
  double2 *Pz = nullptr;
  if (p.splitk > 1) {
    const int64_t kb = (int64_t)blockIdx.z * p.k_chunk;
    Kl = p.K - kb < p.k_chunk ? p.K - kb : p.k_chunk;
    A += kb * p.a_sk;
    B += kb * p.b_sk;
    Pz = static_cast<double2 *>(p.partial) + (int64_t)blockIdx.z * p.M * p.N;
  }
  const bool a_mfast = (p.a_sk != 1), b_nfast = (p.b_sk != 1);
  constexpr int LA = BM * BK / NT, LB = BN * BK / NT;
  float2 ra[LA], rb[LB];
  auto gload = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < LA; i++) {
      const int idx = tid + i * NT;
      int m, k;
      if (a_mfast) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      const int64_t gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < p.M && gk < Kl) ? A[gm * p.a_sm + gk * p.a_sk] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < LB; i++) {
      const int idx = tid + i * NT;
      int n, k;
      if (b_nfast) { k = idx / BN; n = idx % BN; } else { n = idx / BK; k = idx % BK; }
      const int64_t gn = n0 + n, gk = k0 + k;
      rb[i] = (gn < p.N && gk < Kl) ? B[gk * p.b_sk + gn * p.b_sn] : make_float2(0.f, 0.f);
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; i++) {
      const int idx = tid + i * NT;
      int m, k;
      if (a_mfast) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      Ar[buf][k][m] = (double)ra[i].x;
      Ai[buf][k][m] = (double)ra[i].y;
    }
#pragma unroll
    for (int i = 0; i < LB; i++) {
      const int idx = tid + i * NT;
      int n, k;
      if (b_nfast) { k = idx / BN; n = idx % BN; } else { n = idx / BK; k = idx % BK; }
      Br[buf][k][n] = (double)rb[i].x;
      Bi[buf][k][n] = (double)rb[i].y;
    }
  };
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;   // 2 x 4 warps of 32 x 16
  const int fr = lane >> 2, fk = lane & 3;
  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 2; j++) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  const int KT = (int)((Kl + BK - 1) / BK);
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < KT; kt++) {
    const int buf = kt & 1;
    if (kt + 1 < KT) gload((int64_t)(kt + 1) * BK);
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double ar[4], ai[4], nai[4], br[2], bi[2];
#pragma unroll
      for (int i = 0; i < 4; i++) {
        ar[i] = Ar[buf][k4 + fk][wm + 8 * i + fr];
        ai[i] = Ai[buf][k4 + fk][wm + 8 * i + fr];
        nai[i] = -ai[i];
      }
#pragma unroll
      for (int j = 0; j < 2; j++) {
        br[j] = Br[buf][k4 + fk][wn + 8 * j + fr];
        bi[j] = Bi[buf][k4 + fk][wn + 8 * j + fr];
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) {
          dmma884(cr[i][j], ar[i], br[j]);
          dmma884(cr[i][j], nai[i], bi[j]);
          dmma884(ci[i][j], ar[i], bi[j]);
          dmma884(ci[i][j], ai[i], br[j]);
        }
    }
    if (kt + 1 < KT) {
      sstore(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int64_t m = m0 + wm + 8 * i + fr;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t n = n0 + wn + 8 * j + 2 * fk + h;
        if (n >= p.N) continue;
        if (Pz) Pz[m * p.N + n] = make_double2(cr[i][j][h], ci[i][j][h]);
        else C[p.c_row ? p.c_row[m] + p.c_col[n] : m * p.c_sm + n] = make_float2((float)cr[i][j][h], (float)ci[i][j][h]);
      }
  }
}

cudaError_t run_c64_dmma(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  const int64_t tm = (p.M + kCdBM - 1) / kCdBM, tn = (p.N + kCdBN - 1) / kCdBN;
  if (tm * tn > 0x7fffffffLL || p.splitk > 65535) return cudaErrorInvalidConfiguration;
  cudaError_t e = ensure_smem_attr((const void *)gemm_c64_dmma_kernel, cd_smem());
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)(tm * tn), 1, (unsigned)(p.splitk > 1 ? p.splitk : 1));
  gemm_c64_dmma_kernel<<<grid, 256, cd_smem(), s>>>(p, (int)tm, (int)tn);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// TCI_F32_DMMA=0 keeps the SIMT kernel for float32 (A/B)
bool f32_dmma_disabled() {
  static const bool off = [] {
    const char *e = getenv("TCI_F32_DMMA");
    return e && e[0] == '0';
  }();
  return off;
}

template <int BM, int BN>
cudaError_t run_f32_dmma_t(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  const int64_t tm = (p.M + BM - 1) / BM, tn = (p.N + BN - 1) / BN;
  if (tm * tn > 0x7fffffffLL || p.splitk > 65535) return cudaErrorInvalidConfiguration;
  auto k = gemm_f32_dmma_kernel<BM, BN>;
  cudaError_t e = ensure_smem_attr((const void *)k, fd_smem<BM, BN>());
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)(tm * tn), 1, (unsigned)(p.splitk > 1 ? p.splitk : 1));
  k<<<grid, (BM / 32) * (BN / 32) * 32, fd_smem<BM, BN>(), s>>>(p, (int)tm, (int)tn);
  if (launches) ++*launches;
  return cudaGetLastError();
}
cudaError_t run_f32_dmma(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  if (p.N <= 64 && p.M > 64) return run_f32_dmma_t<128, 64>(p, s, launches);
  if (p.M <= 64 && p.N > 64) return run_f32_dmma_t<64, 128>(p, s, launches);
  return run_f32_dmma_t<128, 128>(p, s, launches);
}

template <typename E, int BM, int BN, int BK, int TM, int TN>
cudaError_t run_simt(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  const int64_t tm = (p.M + BM - 1) / BM, tn = (p.N + BN - 1) / BN;
  if (tm * tn > 0x7fffffffLL || p.splitk > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)(tm * tn), 1, (unsigned)(p.splitk > 1 ? p.splitk : 1));
  gemm_simt_kernel<E, BM, BN, BK, TM, TN><<<grid, 256, 0, s>>>(p, (int)tm, (int)tn);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm_f32(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  if (p.dtype == TCI_R32) {
    if (!f32_dmma_disabled()) return run_f32_dmma(p, s, launches);
    // narrow N or M: a 128 x 64 (64 x 128) tile wastes less of the register tile
    if (p.N <= 64 && p.M > 64) return run_simt<float, 128, 64, 8, 8, 4>(p, s, launches);
    if (p.M <= 64 && p.N > 64) return run_simt<float, 64, 128, 8, 4, 8>(p, s, launches);
    return run_simt<float, 128, 128, 8, 8, 8>(p, s, launches);
  }
  if (!f32_dmma_disabled()) return run_c64_dmma(p, s, launches);
  return run_simt<float2, 64, 64, 8, 4, 4>(p, s, launches);
}

}  // namespace tci
