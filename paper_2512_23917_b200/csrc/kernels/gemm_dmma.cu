// gemm_dmma.cu -- GEMM over fused contracted legs:
//   C[m,n] = sum_k A(m,k) B(k,n)          (Eq. (3))
// for float64 and complex128 on the FP64 tensor cores of sm_100a.
//
// sm_100a has no tcgen05 kind for f64 (ptxas rejects .kind::f64) and no
// wgmma, so the FP64 tensor path is the warp-synchronous
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4). Measured on this pool's B200:
// 37.06 TF/s register-resident DMMA peak (profiles/step0_fp64_probe.json).
// At 64 FP64 MAC/clk/SM one DMMA.8x8x4 issues every 16 cycles per SMSP, so
// the kernel is built to keep that pipe busy and nothing else: operands are
// staged global->smem by a 3/4-stage cp.async pipeline (16-byte chunks,
// zero-fill for ragged edges) into padded tiles whose row pitch makes every
// fragment load bank-conflict free (pitch mod 128 B = 32 B for
// 4-rows x 32 B phases, 64 B for 2-rows x 64 B phases), and each warp holds a
// 32x32 (complex) / 64x32 (real) accumulator tile in registers so every
// fragment is reused 4-8 times.
//
// complex128: interleaved (re,im) in global and smem; one LDS.128 yields both
// parts of a fragment element. "4M": Cr += Ar.Br + (-Ai).Bi,
// Ci += Ar.Bi + Ai.Br (two accumulator sets). Each output element is summed
// over k in ascending chunks of 4 (one DMMA), independent of tiling, grid
// size or sharding -> bitwise reproducible across runs and across P
// (R10, R18). No split-K.
#include <cstdio>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

template <bool CPLX, int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, bool A_K_, bool B_K_,
          int VEC_>
struct Cfg {
  static constexpr bool kCplx = CPLX;
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr bool A_K = A_K_, B_K = B_K_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NT = 32 * WARPS_M * WARPS_N;
  static constexpr int ESZ = CPLX ? 16 : 8;               // element bytes
  static constexpr int CHUNK = CPLX ? 1 : VEC_;            // elements per cp.async
  static constexpr int CPB = CHUNK * ESZ;                  // bytes per cp.async
  // padded pitches (elements): see header comment
  static constexpr int PADK = 4;
  static constexpr int PADMN = CPLX ? 2 : 4;
  static constexpr int SA = A_K ? (BK + PADK) : (BM + PADMN);
  static constexpr int SB = B_K ? (BK + PADK) : (BN + PADMN);
  static constexpr int A_STAGE = A_K ? BM * SA : BK * SA;  // elements
  static constexpr int B_STAGE = B_K ? BN * SB : BK * SB;
  static constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) * ESZ;
  static constexpr int MI = WM / 8, NJ = WN / 8;
};

template <class C>
struct Elem {
  using T = typename std::conditional<C::kCplx, double2, double>::type;
};

template <class C>
__device__ __forceinline__ void load_stage(const GemmProblem &p, const char *Ab, const char *Bb,
                                           char *sA, char *sB, int64_t m0, int64_t n0,
                                           int64_t k0) {
  const int tid = threadIdx.x;
  constexpr int ESZ = C::ESZ;
  // ---- A tile ----
  if constexpr (C::A_K) {
    constexpr int CPR = C::BK / C::CHUNK;                 // chunks per row (m)
    constexpr int TOT = C::BM * CPR;
#pragma unroll
    for (int c = tid; c < TOT; c += C::NT) {
      const int m = c / CPR, k = (c % CPR) * C::CHUNK;
      const int64_t gm = m0 + m, gk = k0 + k;
      int valid = 0;
      if (gm < p.M && gk < p.K) valid = (int)min((int64_t)C::CHUNK, p.K - gk);
      const char *src = valid ? Ab + (gm * p.a_sm + gk) * ESZ : Ab;
      cp_async_zfill<C::CPB>(sA + (m * C::SA + k) * ESZ, src, valid * ESZ);
    }
  } else {
    constexpr int CPR = C::BM / C::CHUNK;
    constexpr int TOT = C::BK * CPR;
#pragma unroll
    for (int c = tid; c < TOT; c += C::NT) {
      const int k = c / CPR, m = (c % CPR) * C::CHUNK;
      const int64_t gm = m0 + m, gk = k0 + k;
      int valid = 0;
      if (gm < p.M && gk < p.K) valid = (int)min((int64_t)C::CHUNK, p.M - gm);
      const char *src = valid ? Ab + (gk * p.a_sk + gm) * ESZ : Ab;
      cp_async_zfill<C::CPB>(sA + (k * C::SA + m) * ESZ, src, valid * ESZ);
    }
  }
  // ---- B tile ----
  if constexpr (C::B_K) {
    constexpr int CPR = C::BK / C::CHUNK;
    constexpr int TOT = C::BN * CPR;
#pragma unroll
    for (int c = tid; c < TOT; c += C::NT) {
      const int n = c / CPR, k = (c % CPR) * C::CHUNK;
      const int64_t gn = n0 + n, gk = k0 + k;
      int valid = 0;
      if (gn < p.N && gk < p.K) valid = (int)min((int64_t)C::CHUNK, p.K - gk);
      const char *src = valid ? Bb + (gn * p.b_sn + gk) * ESZ : Bb;
      cp_async_zfill<C::CPB>(sB + (n * C::SB + k) * ESZ, src, valid * ESZ);
    }
  } else {
    constexpr int CPR = C::BN / C::CHUNK;
    constexpr int TOT = C::BK * CPR;
#pragma unroll
    for (int c = tid; c < TOT; c += C::NT) {
      const int k = c / CPR, n = (c % CPR) * C::CHUNK;
      const int64_t gn = n0 + n, gk = k0 + k;
      int valid = 0;
      if (gn < p.N && gk < p.K) valid = (int)min((int64_t)C::CHUNK, p.N - gn);
      const char *src = valid ? Bb + (gk * p.b_sk + gn) * ESZ : Bb;
      cp_async_zfill<C::CPB>(sB + (k * C::SB + n) * ESZ, src, valid * ESZ);
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1) gemm_dmma_kernel(const GemmProblem p, int tiles_m,
                                                             int tiles_n) {
  using T = typename Elem<C>::T;
  extern __shared__ __align__(128) char smem[];
  char *sA0 = smem;
  char *sB0 = smem + C::STAGES * C::A_STAGE * C::ESZ;

  // grouped rasterization: 8 M-tiles share the B panels in L2
  constexpr int GROUP = 8;
  const int bid = blockIdx.x;
  const int per_group = GROUP * tiles_n;
  const int first_m = (bid / per_group) * GROUP;
  const int gsize = min(tiles_m - first_m, GROUP);
  const int tile_m = first_m + (bid % per_group) % gsize;
  const int tile_n = (bid % per_group) / gsize;
  const int64_t m0 = (int64_t)tile_m * C::BM, n0 = (int64_t)tile_n * C::BN;

  const int64_t bz = blockIdx.z;
  const char *Ab = static_cast<const char *>(p.A) + bz * p.a_sb * C::ESZ;
  const char *Bb = static_cast<const char *>(p.B) + bz * p.b_sb * C::ESZ;
  char *Cb = static_cast<char *>(p.C) + bz * p.c_sb * C::ESZ;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / C::WARPS_N) * C::WM, wn0 = (warp % C::WARPS_N) * C::WN;
  const int lr = lane >> 2, lc = lane & 3;

  double accr[C::MI][C::NJ][2];
  double acci[C::kCplx ? C::MI : 1][C::kCplx ? C::NJ : 1][2];
#pragma unroll
  for (int i = 0; i < C::MI; i++)
#pragma unroll
    for (int j = 0; j < C::NJ; j++) accr[i][j][0] = accr[i][j][1] = 0.0;
  if constexpr (C::kCplx) {
#pragma unroll
    for (int i = 0; i < C::MI; i++)
#pragma unroll
      for (int j = 0; j < C::NJ; j++) acci[i][j][0] = acci[i][j][1] = 0.0;
  }

  const int KT = (int)((p.K + C::BK - 1) / C::BK);
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; s++) {
    if (s < KT)
      load_stage<C>(p, Ab, Bb, sA0 + s * C::A_STAGE * C::ESZ, sB0 + s * C::B_STAGE * C::ESZ, m0,
                    n0, (int64_t)s * C::BK);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; kt++) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + C::STAGES - 1;
      if (nk < KT) {
        const int st = nk % C::STAGES;
        load_stage<C>(p, Ab, Bb, sA0 + st * C::A_STAGE * C::ESZ, sB0 + st * C::B_STAGE * C::ESZ,
                      m0, n0, (int64_t)nk * C::BK);
      }
      cp_async_commit();
    }
    const int st = kt % C::STAGES;
    const T *sA = reinterpret_cast<const T *>(sA0 + st * C::A_STAGE * C::ESZ);
    const T *sB = reinterpret_cast<const T *>(sB0 + st * C::B_STAGE * C::ESZ);
#pragma unroll
    for (int kk = 0; kk < C::BK / 4; kk++) {
      const int k = kk * 4 + lc;
      T af[C::MI], bf[C::NJ];
#pragma unroll
      for (int i = 0; i < C::MI; i++) {
        const int m = wm0 + i * 8 + lr;
        af[i] = C::A_K ? sA[m * C::SA + k] : sA[k * C::SA + m];
      }
#pragma unroll
      for (int j = 0; j < C::NJ; j++) {
        const int n = wn0 + j * 8 + lr;
        bf[j] = C::B_K ? sB[n * C::SB + k] : sB[k * C::SB + n];
      }
      if constexpr (C::kCplx) {
#pragma unroll
        for (int i = 0; i < C::MI; i++) {
          const double ar = af[i].x, ai = af[i].y, nai = -af[i].y;
#pragma unroll
          for (int j = 0; j < C::NJ; j++) {
            dmma884(accr[i][j], ar, bf[j].x);
            dmma884(acci[i][j], ar, bf[j].y);
            dmma884(accr[i][j], nai, bf[j].y);
            dmma884(acci[i][j], ai, bf[j].x);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < C::MI; i++)
#pragma unroll
          for (int j = 0; j < C::NJ; j++) dmma884(accr[i][j], af[i], bf[j]);
      }
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: C N-contiguous, direct 16-byte stores ----
#pragma unroll
  for (int i = 0; i < C::MI; i++) {
    const int64_t m = m0 + wm0 + i * 8 + lr;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < C::NJ; j++) {
      const int64_t n = n0 + wn0 + j * 8 + 2 * lc;
      if constexpr (C::kCplx) {
        double2 *cp = reinterpret_cast<double2 *>(Cb) + m * p.c_sm + n;
        if (n < p.N) cp[0] = make_double2(accr[i][j][0], acci[i][j][0]);
        if (n + 1 < p.N) cp[1] = make_double2(accr[i][j][1], acci[i][j][1]);
      } else {
        double *cp = reinterpret_cast<double *>(Cb) + m * p.c_sm + n;
        if (n < p.N) cp[0] = accr[i][j][0];
        if (n + 1 < p.N) cp[1] = accr[i][j][1];
      }
    }
  }
}

template <class C>
cudaError_t run(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  auto kern = gemm_dmma_kernel<C>;
  static uint64_t attr_set = 0;   // per instantiation, one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set >> dev & 1)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set |= 1ull << dev;
  }
  const int64_t tm = (p.M + C::BM - 1) / C::BM, tn = (p.N + C::BN - 1) / C::BN;
  if (tm * tn > 0x7fffffffLL || p.batch > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)(tm * tn), 1, (unsigned)p.batch);
  kern<<<grid, C::NT, C::SMEM, s>>>(p, (int)tm, (int)tn);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// complex128: CTA 64x128, BK 8, 8 warps of 32x32, 4 stages (96 KB smem)
template <bool AK, bool BK>
using ZCfg = Cfg<true, 64, 128, 8, 32, 32, 4, AK, BK, 1>;
// float64: CTA 128x128, BK 16, 8 warps of 64x32, 3 stages
template <bool AK, bool BK, int VEC>
using DCfg = Cfg<false, 128, 128, 16, 64, 32, 3, AK, BK, VEC>;

}  // namespace

cudaError_t launch_gemm_f32(const GemmProblem &p, cudaStream_t s, int64_t *launches);

cudaError_t launch_gemm(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  if (p.M == 0 || p.N == 0) return cudaSuccess;
  if (p.dtype == TCI_R32 || p.dtype == TCI_C64) return launch_gemm_f32(p, s, launches);
  // The planner canonicalises strides (plan.cpp, canonical_gemm): a_sk == 1
  // selects the K-contiguous loader, otherwise a_sm == 1; same for B.
  const bool ak = (p.a_sk == 1), bk = (p.b_sk == 1);
  if (p.dtype == TCI_C128) {
    if (ak && bk) return run<ZCfg<true, true>>(p, s, launches);
    if (ak && !bk) return run<ZCfg<true, false>>(p, s, launches);
    if (!ak && bk) return run<ZCfg<false, true>>(p, s, launches);
    return run<ZCfg<false, false>>(p, s, launches);
  }
  // float64: 16-byte chunks need 16-byte aligned rows
  const int64_t lda = ak ? p.a_sm : p.a_sk, ldb = bk ? p.b_sn : p.b_sk;
  const bool aligned = ((uintptr_t)p.A % 16 == 0) && ((uintptr_t)p.B % 16 == 0) &&
                       (lda % 2 == 0 || (ak ? p.M : p.K) == 1) &&
                       (ldb % 2 == 0 || (bk ? p.N : p.K) == 1) && (p.a_sb % 2 == 0) &&
                       (p.b_sb % 2 == 0);
  if (aligned) {
    if (ak && bk) return run<DCfg<true, true, 2>>(p, s, launches);
    if (ak && !bk) return run<DCfg<true, false, 2>>(p, s, launches);
    if (!ak && bk) return run<DCfg<false, true, 2>>(p, s, launches);
    return run<DCfg<false, false, 2>>(p, s, launches);
  }
  if (ak && bk) return run<DCfg<true, true, 1>>(p, s, launches);
  if (ak && !bk) return run<DCfg<true, false, 1>>(p, s, launches);
  if (!ak && bk) return run<DCfg<false, true, 1>>(p, s, launches);
  return run<DCfg<false, false, 1>>(p, s, launches);
}

}  // namespace tci
