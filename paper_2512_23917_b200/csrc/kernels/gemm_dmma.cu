// gemm_dmma.cu -- GEMM over fused contracted legs:
//   C[m,n] = sum_k A(m,k) B(k,n)          (Eq. (3))
// for float64 and complex128 on the FP64 tensor cores of sm_100a.
//
// sm_100a has no tcgen05 kind for f64 (ptxas rejects .kind::f64) and no
// wgmma, so the FP64 tensor path is the warp-synchronous
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4). Measured on this pool's B200
// (profiles/step0_*): 37.06 TF/s DMMA peak, 36.7 TF/s DFMA peak, and DMMA +
// DFMA together never exceed ~37 TF/s -- one FP64 datapath. The only way to
// run a complex GEMM faster than the 4-real-product rate is to do fewer real
// products:
//
// complex128, "3M" (Gauss): with P = Ar.Br, Q = Ai.Bi, S = (Ar+Ai).(Br+Bi),
//   Cr = P - Q,  Ci = S - P - Q
// -- 3 DMMAs per complex fragment product instead of 4 (the sums cost one
// DADD per fragment element, ~1/64 of the DMMA work). Error is normwise
// (|Ci error| <~ K u (|Ar|+|Ai|)(|Br|+|Bi|)), inside the 1e-12 relative-
// Frobenius parity bar (R11). A 4M variant (Cr += Ar.Br - Ai.Bi,
// Ci += Ar.Bi + Ai.Br) is kept and selectable (tci_set_gemm_algorithm).
//
// Kernel structure (one CTA per 64x64 complex / 128x128 real output tile):
//  * 6-stage (complex) / 3-stage (real) cp.async pipeline, 16-byte chunks, zero-fill on ragged edges;
//    each thread's chunk pointers and row predicates are computed once and
//    advanced by a constant per K tile (no per-tile 64-bit index math);
//  * padded shared-memory pitches make every fragment load conflict free
//    (pitch mod 128 B = 32 B for 4-row x 32 B phases, 64 B for 2 x 64 B);
//  * fragments are double-buffered in registers: the next k-step's (or the
//    next stage's first) fragments are loaded before the current DMMAs
//    issue, so DMMA never waits on a shared-memory load;
//  * each output element is summed over k in ascending chunks of 4 (one
//    DMMA) for every tiling, grid size and shard -> bitwise reproducible
//    across runs and across P (R10, R18). No split-K.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>

#include "../tci_internal.h"
#include "common.cuh"

// tools/gemm_lab.cu may redefine this to measure the cost of the 3M sums
#ifndef TCI_LAB_SUM
#define TCI_LAB_SUM(x, y) ((x) + (y))
#endif

namespace tci {
namespace {

enum Algo { kReal = 0, kCplx3M = 1, kCplx4M = 2, kCplx3MS = 3 };
// kCplx3MS: 3M with the (re+im) sums formed once per CTA per stage into a
// shared-memory sum plane (each thread sums the chunks it loaded), instead
// of once per warp per fragment in registers

template <int ALGO, int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, bool A_K_, bool B_K_,
          int VEC_, int MODE_ = 0>
struct Cfg {
  static constexpr int kAlgo = ALGO;
  static constexpr int MODE = MODE_;   // 0 plain GEMM, 1 TEBD theta (gate in the epilogue)
  static constexpr bool kCplx = ALGO != kReal;
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr bool A_K = A_K_, B_K = B_K_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NT = 32 * WARPS_M * WARPS_N;
  static constexpr int ESZ = kCplx ? 16 : 8;               // element bytes
  static constexpr int CHUNK = kCplx ? 1 : VEC_;            // elements per cp.async
  static constexpr int CPB = CHUNK * ESZ;                   // bytes per cp.async
  static constexpr int PADK = 4;
  static constexpr int PADMN = kCplx ? 2 : 4;
  static constexpr int SA = A_K ? (BK + PADK) : (BM + PADMN);
  static constexpr int SB = B_K ? (BK + PADK) : (BN + PADMN);
  static constexpr int A_STAGE = A_K ? BM * SA : BK * SA;   // elements
  static constexpr int B_STAGE = B_K ? BN * SB : BK * SB;
  static constexpr bool kSumPlane = ALGO == kCplx3MS;
  static constexpr int SPA = A_K ? (BK + 4) : (BM + 4);     // sum-plane pitches (doubles)
  static constexpr int SPB = B_K ? (BK + 4) : (BN + 4);
  static constexpr int A_SUM = kSumPlane ? (A_K ? BM * SPA : BK * SPA) : 0;   // doubles per stage
  static constexpr int B_SUM = kSumPlane ? (B_K ? BN * SPB : BK * SPB) : 0;
  static constexpr int SMEM_PIPE = STAGES * (A_STAGE + B_STAGE) * ESZ + STAGES * (A_SUM + B_SUM) * 8;
  static constexpr int SMEM_EPI = MODE == 1 ? BM * (BN + 1) * 8 : 0;   // staged C tile (TEBD)
  static constexpr int SMEM = SMEM_PIPE > SMEM_EPI ? SMEM_PIPE : SMEM_EPI;
  static constexpr int MI = WM / 8, NJ = WN / 8;
  static constexpr int KK = BK / 4;
  // loader geometry: chunks per tile row along the contiguous leg
  static constexpr int A_CPR = A_K ? BK / CHUNK : BM / CHUNK;
  static constexpr int A_ROWS = A_K ? BM : BK;
  static constexpr int A_PER_T = A_ROWS * A_CPR / NT;
  static constexpr int B_CPR = B_K ? BK / CHUNK : BN / CHUNK;
  static constexpr int B_ROWS = B_K ? BN : BK;
  static constexpr int B_PER_T = B_ROWS * B_CPR / NT;
  static_assert(A_ROWS * A_CPR % NT == 0 && B_ROWS * B_CPR % NT == 0, "loader split");
  static_assert(NT % A_CPR == 0 && NT % B_CPR == 0, "loader rows");
};

// One operand's per-thread loader state. The tile is ROWS rows of CPR chunks
// along the operand's contiguous leg; thread t owns chunk column (t % CPR)
// of rows t / CPR + i * (NT / CPR).
template <class C, bool IS_A>
struct Loader {
  static constexpr bool KMAJ = IS_A ? C::A_K : C::B_K;
  static constexpr int CPR = IS_A ? C::A_CPR : C::B_CPR;
  static constexpr int PER_T = IS_A ? C::A_PER_T : C::B_PER_T;
  static constexpr int RSTEP = C::NT / CPR;
  static constexpr int S = IS_A ? C::SA : C::SB;
  const char *base;           // operand base (a valid dummy address)
  const char *ptr[PER_T];     // global address of this thread's chunk in K tile 0
  uint32_t soff[PER_T];       // byte offset inside a stage
  int kidx[PER_T];            // k index (within the tile) of the chunk's first element
  int nvalid_mn[PER_T];       // K-major: row valid (0/1); MN-major: valid elements in the chunk
  int64_t kstep;              // bytes to advance per K tile
  uint32_t sumoff[PER_T];     // element offset of this chunk in the stage's sum plane

  __device__ __forceinline__ void set_sum_offsets() {
    if constexpr (C::kSumPlane) {
      constexpr int SP = IS_A ? C::SPA : C::SPB;
      const int t = threadIdx.x;
      const int col = (t % CPR) * C::CHUNK;
#pragma unroll
      for (int i = 0; i < PER_T; i++) sumoff[i] = (uint32_t)((t / CPR + i * RSTEP) * SP + col);
    }
  }
  // (re + im) of this thread's landed chunks of one stage into its sum plane
  __device__ __forceinline__ void make_sums(const char *stage, double *sums) const {
    if constexpr (C::kSumPlane) {
#pragma unroll
      for (int i = 0; i < PER_T; i++) {
        const double2 v = *reinterpret_cast<const double2 *>(stage + soff[i]);
        sums[sumoff[i]] = TCI_LAB_SUM(v.x, v.y);
      }
    }
  }

  // s_mn / s_k: element strides of the M (or N) and K legs
  __device__ __forceinline__ void init(const char *b, int64_t mn0, int64_t MN, int64_t s_mn,
                                       int64_t s_k) {
    base = b;
    const int t = threadIdx.x;
    const int col = (t % CPR) * C::CHUNK;
#pragma unroll
    for (int i = 0; i < PER_T; i++) {
      const int row = t / CPR + i * RSTEP;
      if (KMAJ) {   // rows are m (or n), chunk columns are k
        const int64_t g = mn0 + row;
        nvalid_mn[i] = g < MN ? 1 : 0;
        kidx[i] = col;
        ptr[i] = b + ((g < MN ? g : 0) * s_mn + col) * C::ESZ;
      } else {      // rows are k, chunk columns are m (or n)
        const int64_t g = mn0 + col;
        nvalid_mn[i] = (int)(g < MN ? (MN - g < C::CHUNK ? MN - g : C::CHUNK) : 0);
        kidx[i] = row;
        ptr[i] = b + ((int64_t)row * s_k + (g < MN ? g : 0)) * C::ESZ;
      }
      soff[i] = (uint32_t)((row * S + col) * C::ESZ);
    }
    kstep = (int64_t)C::BK * (KMAJ ? 1 : s_k) * C::ESZ;
  }

  // TEBD A (K-major): tile row r holds (a, s) = (a0 + r / 2, r % 2)
  __device__ __forceinline__ void init_tebd_a(const char *b, int64_t a0, int64_t chi_a, int64_t s_a,
                                              int64_t s_s) {
    base = b;
    const int t = threadIdx.x;
    const int col = (t % CPR) * C::CHUNK;
#pragma unroll
    for (int i = 0; i < PER_T; i++) {
      const int row = t / CPR + i * RSTEP;
      const int64_t a = a0 + row / 2;
      nvalid_mn[i] = a < chi_a ? 1 : 0;
      kidx[i] = col;
      ptr[i] = b + ((a < chi_a ? a : 0) * s_a + (row % 2) * s_s + col) * C::ESZ;
      soff[i] = (uint32_t)((row * S + col) * C::ESZ);
    }
    kstep = (int64_t)C::BK * C::ESZ;
  }
  // TEBD B (N-major): tile column l holds (t, c) = (l / (BN/2), c0 + l % (BN/2))
  __device__ __forceinline__ void init_tebd_b(const char *b, int64_t c0, int64_t chi_c, int64_t s_k,
                                              int64_t s_t) {
    base = b;
    const int t = threadIdx.x;
    const int col = (t % CPR) * C::CHUNK;
    constexpr int HALF = C::BN / 2;
    const int64_t c = c0 + col % HALF;
#pragma unroll
    for (int i = 0; i < PER_T; i++) {
      const int row = t / CPR + i * RSTEP;
      nvalid_mn[i] = (int)(c < chi_c ? (chi_c - c < C::CHUNK ? chi_c - c : C::CHUNK) : 0);
      kidx[i] = row;
      ptr[i] = b + ((int64_t)row * s_k + (col / HALF) * s_t + (c < chi_c ? c : 0)) * C::ESZ;
      soff[i] = (uint32_t)((row * S + col) * C::ESZ);
    }
    kstep = (int64_t)C::BK * s_k * C::ESZ;
  }

  // issue this thread's cp.asyncs for K tile kt into the stage at `sbase`
  __device__ __forceinline__ void load(char *sbase, int kt, int64_t K, bool full_k) const {
    const int64_t k0 = (int64_t)kt * C::BK;
#pragma unroll
    for (int i = 0; i < PER_T; i++) {
      int bytes;
      if (KMAJ) {
        int nk = C::CHUNK;
        if (!full_k) {
          const int64_t rem = K - (k0 + kidx[i]);
          nk = rem <= 0 ? 0 : (rem < C::CHUNK ? (int)rem : C::CHUNK);
        }
        bytes = nvalid_mn[i] ? nk * C::ESZ : 0;
      } else {
        const bool kok = full_k || (k0 + kidx[i] < K);
        bytes = kok ? nvalid_mn[i] * C::ESZ : 0;
      }
      const char *src = bytes ? ptr[i] + kt * kstep : base;   // nothing is read when bytes == 0
      cp_async_zfill<C::CPB>(sbase + soff[i], src, bytes);
    }
  }
};

template <class C>
struct Frag {
  // complex 3M: (re, im, re+im) per fragment element; 4M: (re, im); real: 1
  static constexpr int NV = (C::kAlgo == kCplx3M || C::kAlgo == kCplx3MS) ? 3 : (C::kCplx ? 2 : 1);
  double a[C::MI][NV], b[C::NJ][NV];
};

template <class C>
__device__ __forceinline__ void load_frag(Frag<C> &f, const char *sA, const char *sB, int kk,
                                          int wm0, int wn0, int lr, int lc,
                                          const double *sumA = nullptr, const double *sumB = nullptr) {
  const int k = kk * 4 + lc;
  if constexpr (C::kSumPlane) {
    const double2 *A = reinterpret_cast<const double2 *>(sA);
    const double2 *B = reinterpret_cast<const double2 *>(sB);
#pragma unroll
    for (int i = 0; i < C::MI; i++) {
      const int m = wm0 + i * 8 + lr;
      const double2 v = C::A_K ? A[m * C::SA + k] : A[k * C::SA + m];
      f.a[i][0] = v.x;
      f.a[i][1] = v.y;
      f.a[i][2] = C::A_K ? sumA[m * C::SPA + k] : sumA[k * C::SPA + m];
    }
#pragma unroll
    for (int j = 0; j < C::NJ; j++) {
      const int n = wn0 + j * 8 + lr;
      const double2 v = C::B_K ? B[n * C::SB + k] : B[k * C::SB + n];
      f.b[j][0] = v.x;
      f.b[j][1] = v.y;
      f.b[j][2] = C::B_K ? sumB[n * C::SPB + k] : sumB[k * C::SPB + n];
    }
  } else if constexpr (C::kCplx) {
    const double2 *A = reinterpret_cast<const double2 *>(sA);
    const double2 *B = reinterpret_cast<const double2 *>(sB);
#pragma unroll
    for (int i = 0; i < C::MI; i++) {
      const int m = wm0 + i * 8 + lr;
      const double2 v = C::A_K ? A[m * C::SA + k] : A[k * C::SA + m];
      f.a[i][0] = v.x;
      f.a[i][1] = v.y;
      if constexpr (C::kAlgo == kCplx3M) f.a[i][2] = TCI_LAB_SUM(v.x, v.y);
    }
#pragma unroll
    for (int j = 0; j < C::NJ; j++) {
      const int n = wn0 + j * 8 + lr;
      const double2 v = C::B_K ? B[n * C::SB + k] : B[k * C::SB + n];
      f.b[j][0] = v.x;
      f.b[j][1] = v.y;
      if constexpr (C::kAlgo == kCplx3M) f.b[j][2] = TCI_LAB_SUM(v.x, v.y);
    }
  } else {
    const double *A = reinterpret_cast<const double *>(sA);
    const double *B = reinterpret_cast<const double *>(sB);
#pragma unroll
    for (int i = 0; i < C::MI; i++) {
      const int m = wm0 + i * 8 + lr;
      f.a[i][0] = C::A_K ? A[m * C::SA + k] : A[k * C::SA + m];
    }
#pragma unroll
    for (int j = 0; j < C::NJ; j++) {
      const int n = wn0 + j * 8 + lr;
      f.b[j][0] = C::B_K ? B[n * C::SB + k] : B[k * C::SB + n];
    }
  }
}

template <class C>
struct Acc {
  static constexpr int NS = (C::kAlgo == kCplx3M || C::kAlgo == kCplx3MS) ? 3 : (C::kCplx ? 2 : 1);
  double c[NS][C::MI][C::NJ][2];
};

template <class C>
__device__ __forceinline__ void mma_step(Acc<C> &acc, const Frag<C> &f) {
#pragma unroll
  for (int i = 0; i < C::MI; i++)
#pragma unroll
    for (int j = 0; j < C::NJ; j++) {
      if constexpr (C::kAlgo == kCplx3M || C::kAlgo == kCplx3MS) {
        dmma884(acc.c[0][i][j], f.a[i][0], f.b[j][0]);   // P = Ar.Br
        dmma884(acc.c[1][i][j], f.a[i][1], f.b[j][1]);   // Q = Ai.Bi
        dmma884(acc.c[2][i][j], f.a[i][2], f.b[j][2]);   // S = (Ar+Ai).(Br+Bi)
      } else if constexpr (C::kAlgo == kCplx4M) {
        dmma884(acc.c[0][i][j], f.a[i][0], f.b[j][0]);
        dmma884(acc.c[1][i][j], f.a[i][0], f.b[j][1]);
        dmma884(acc.c[0][i][j], -f.a[i][1], f.b[j][1]);
        dmma884(acc.c[1][i][j], f.a[i][1], f.b[j][0]);
      } else {
        dmma884(acc.c[0][i][j], f.a[i][0], f.b[j][0]);
      }
    }
}

// one output tile (grid position bid) of the GEMM
template <class C>
__device__ __forceinline__ void gemm_dmma_tile(const GemmProblem &p, int tiles_m, int tiles_n, int bid, char *smem) {
  char *sA0 = smem;
  char *sB0 = smem + C::STAGES * C::A_STAGE * C::ESZ;
  double *sumA0 = reinterpret_cast<double *>(smem + C::STAGES * (C::A_STAGE + C::B_STAGE) * C::ESZ);
  double *sumB0 = sumA0 + C::STAGES * C::A_SUM;

  // grouped rasterization: GROUP M-tiles walk the N-tiles together so the
  // B panels they share stay in L2
  constexpr int GROUP = 8;
  const int per_group = GROUP * tiles_n;
  const int first_m = (bid / per_group) * GROUP;
  const int gsize = min(tiles_m - first_m, GROUP);
  const int tile_m = first_m + (bid % per_group) % gsize;
  const int tile_n = (bid % per_group) / gsize;
  const int64_t m0 = (int64_t)tile_m * C::BM, n0 = (int64_t)tile_n * C::BN;

  const char *Ab = static_cast<const char *>(p.A);
  const char *Bb = static_cast<const char *>(p.B);
  char *Cb = static_cast<char *>(p.C);
  int64_t Kl = p.K, c_sm = p.c_sm;   // this CTA's K extent and C row stride
  if (p.splitk > 1) {
    const int64_t kb = (int64_t)blockIdx.z * p.k_chunk;
    Kl = p.K - kb < p.k_chunk ? p.K - kb : p.k_chunk;
    Ab += kb * p.a_sk * C::ESZ;
    Bb += kb * p.b_sk * C::ESZ;
    Cb = static_cast<char *>(p.partial) + (int64_t)blockIdx.z * p.M * p.N * C::ESZ;
    c_sm = p.N;
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / C::WARPS_N) * C::WM, wn0 = (warp % C::WARPS_N) * C::WN;
  const int lr = lane >> 2, lc = lane & 3;

  Loader<C, true> la;
  Loader<C, false> lb;
  if constexpr (C::MODE == 1) {
    la.init_tebd_a(Ab, (int64_t)tile_m * (C::BM / 2), p.te_chi_a, p.te_a_a, p.te_a_s);
    lb.init_tebd_b(Bb, (int64_t)tile_n * (C::BN / 2), p.te_chi_c, p.b_sk, p.te_b_t);
  } else {
    if (C::A_K) la.init(Ab, m0, p.M, p.a_sm, 1);
    else la.init(Ab, m0, p.M, 1, p.a_sk);
    if (C::B_K) lb.init(Bb, n0, p.N, p.b_sn, 1);
    else lb.init(Bb, n0, p.N, 1, p.b_sk);
  }

  la.set_sum_offsets();
  lb.set_sum_offsets();

  Acc<C> acc;
#pragma unroll
  for (int s = 0; s < Acc<C>::NS; s++)
#pragma unroll
    for (int i = 0; i < C::MI; i++)
#pragma unroll
      for (int j = 0; j < C::NJ; j++) acc.c[s][i][j][0] = acc.c[s][i][j][1] = 0.0;

  const int KT = (int)((Kl + C::BK - 1) / C::BK);
  const int KT_full = (int)(Kl / C::BK);    // tiles with no K tail
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; s++) {
    if (s < KT) {
      la.load(sA0 + s * C::A_STAGE * C::ESZ, s, Kl, s < KT_full);
      lb.load(sB0 + s * C::B_STAGE * C::ESZ, s, Kl, s < KT_full);
    }
    cp_async_commit();
  }
  cp_async_wait<C::STAGES - 2>();
  la.make_sums(sA0, sumA0);
  lb.make_sums(sB0, sumB0);
  __syncthreads();

  Frag<C> fr[2];
  load_frag<C>(fr[0], sA0, sB0, 0, wm0, wn0, lr, lc, sumA0, sumB0);

  for (int kt = 0; kt < KT; kt++) {
    const int st = kt % C::STAGES;
    const char *sA = sA0 + st * C::A_STAGE * C::ESZ;
    const char *sB = sB0 + st * C::B_STAGE * C::ESZ;
    const double *smA = sumA0 + st * C::A_SUM, *smB = sumB0 + st * C::B_SUM;
#pragma unroll
    for (int kk = 0; kk < C::KK; kk++) {
      if (kk < C::KK - 1) {
        load_frag<C>(fr[(kk + 1) & 1], sA, sB, kk + 1, wm0, wn0, lr, lc, smA, smB);
      } else {
        // stage kt+1 must have landed; stage kt-1 is free for reuse
        cp_async_wait<C::STAGES - 3>();
        if (kt + 1 < KT) {
          const int s1 = (kt + 1) % C::STAGES;
          la.make_sums(sA0 + s1 * C::A_STAGE * C::ESZ, sumA0 + s1 * C::A_SUM);
          lb.make_sums(sB0 + s1 * C::B_STAGE * C::ESZ, sumB0 + s1 * C::B_SUM);
        }
        __syncthreads();
        const int nk = kt + C::STAGES - 1;
        if (nk < KT) {
          const int ns = nk % C::STAGES;
          la.load(sA0 + ns * C::A_STAGE * C::ESZ, nk, Kl, nk < KT_full);
          lb.load(sB0 + ns * C::B_STAGE * C::ESZ, nk, Kl, nk < KT_full);
        }
        cp_async_commit();
        if (kt + 1 < KT) {
          const int s1 = (kt + 1) % C::STAGES;
          load_frag<C>(fr[(kk + 1) & 1], sA0 + s1 * C::A_STAGE * C::ESZ,
                       sB0 + s1 * C::B_STAGE * C::ESZ, 0, wm0, wn0, lr, lc, sumA0 + s1 * C::A_SUM,
                       sumB0 + s1 * C::B_SUM);
        }
      }
      mma_step<C>(acc, fr[kk & 1]);
    }
  }
  cp_async_wait<0>();

  if constexpr (C::MODE == 1) {
    // ---- TEBD epilogue: theta[a,p,q,c] = sum_{s,t} U[p,q,s,t] C[(a,s),(t,c)].
    // The CTA holds all (s,t) of its 64 a's x 64 c's; stage C in shared
    // memory, then each thread applies the 4x4 gate to one (a,c) pair and
    // writes its 4 outputs (consecutive threads -> consecutive c).
    __syncthreads();   // pipeline buffers are dead: reuse them for the C tile
    double *Cs = reinterpret_cast<double *>(smem);
    constexpr int PC = C::BN + 1;
#pragma unroll
    for (int i = 0; i < C::MI; i++)
#pragma unroll
      for (int j = 0; j < C::NJ; j++) {
        const int m = wm0 + i * 8 + lr, n = wn0 + j * 8 + 2 * lc;
        Cs[m * PC + n] = acc.c[0][i][j][0];
        Cs[m * PC + n + 1] = acc.c[0][i][j][1];
      }
    double u[2][2][2][2];
#pragma unroll
    for (int pp = 0; pp < 2; pp++)
#pragma unroll
      for (int q = 0; q < 2; q++)
#pragma unroll
        for (int s_ = 0; s_ < 2; s_++)
#pragma unroll
          for (int t_ = 0; t_ < 2; t_++)
            u[pp][q][s_][t_] = p.te_U[pp * p.te_u[0] + q * p.te_u[1] + s_ * p.te_u[2] + t_ * p.te_u[3]];
    __syncthreads();
    constexpr int HA = C::BM / 2, HC = C::BN / 2;
    for (int idx = threadIdx.x; idx < HA * HC; idx += C::NT) {
      const int al = idx / HC, cl = idx % HC;
      const int64_t a = (int64_t)tile_m * HA + al, c = (int64_t)tile_n * HC + cl;
      if (a >= p.te_chi_a || c >= p.te_chi_c) continue;
      double x[2][2];
#pragma unroll
      for (int s_ = 0; s_ < 2; s_++)
#pragma unroll
        for (int t_ = 0; t_ < 2; t_++) x[s_][t_] = Cs[(2 * al + s_) * PC + t_ * HC + cl];
      double *T = p.te_T + a * p.te_t[0] + c * p.te_t[3];
#pragma unroll
      for (int pp = 0; pp < 2; pp++)
#pragma unroll
        for (int q = 0; q < 2; q++) {
          double th = 0.0;
#pragma unroll
          for (int s_ = 0; s_ < 2; s_++)
#pragma unroll
            for (int t_ = 0; t_ < 2; t_++) th = fma(u[pp][q][s_][t_], x[s_][t_], th);
          T[pp * p.te_t[1] + q * p.te_t[2]] = th;
        }
    }
    return;
  }

  // ---- epilogue: C N-contiguous, direct stores (each quad of lanes writes a
  // contiguous 64 B (real) / 128 B (complex) run), or the gamma-order
  // scatter through the row / column offset tables (8(a6)) ----
  const bool scat = p.c_row != nullptr && p.splitk <= 1;
#pragma unroll
  for (int i = 0; i < C::MI; i++) {
    const int64_t m = m0 + wm0 + i * 8 + lr;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < C::NJ; j++) {
      const int64_t n = n0 + wn0 + j * 8 + 2 * lc;
      if constexpr (C::kCplx) {
        double2 *cp = reinterpret_cast<double2 *>(Cb) + m * c_sm + n;
        double2 *cp1 = cp + 1;
        if (scat) {
          cp = reinterpret_cast<double2 *>(Cb) + p.c_row[m] + p.c_col[n];
          if (n + 1 < p.N) cp1 = reinterpret_cast<double2 *>(Cb) + p.c_row[m] + p.c_col[n + 1];
        }
        double re0, im0, re1, im1;
        if constexpr (C::kAlgo == kCplx3M || C::kAlgo == kCplx3MS) {
          const double P0 = acc.c[0][i][j][0], Q0 = acc.c[1][i][j][0], S0 = acc.c[2][i][j][0];
          const double P1 = acc.c[0][i][j][1], Q1 = acc.c[1][i][j][1], S1 = acc.c[2][i][j][1];
          re0 = P0 - Q0;
          im0 = S0 - P0 - Q0;
          re1 = P1 - Q1;
          im1 = S1 - P1 - Q1;
        } else {
          re0 = acc.c[0][i][j][0];
          im0 = acc.c[1][i][j][0];
          re1 = acc.c[0][i][j][1];
          im1 = acc.c[1][i][j][1];
        }
        if (n < p.N) cp[0] = make_double2(re0, im0);
        if (n + 1 < p.N) cp1[0] = make_double2(re1, im1);
      } else {
        double *cp = reinterpret_cast<double *>(Cb) + m * c_sm + n;
        double *cp1 = cp + 1;
        if (scat) {
          cp = reinterpret_cast<double *>(Cb) + p.c_row[m] + p.c_col[n];
          if (n + 1 < p.N) cp1 = reinterpret_cast<double *>(Cb) + p.c_row[m] + p.c_col[n + 1];
        }
        if (n < p.N) cp[0] = acc.c[0][i][j][0];
        if (n + 1 < p.N) cp1[0] = acc.c[0][i][j][1];
      }
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1) gemm_dmma_kernel(const GemmProblem p, int tiles_m, int tiles_n) {
  extern __shared__ __align__(128) char smem[];
  if (!p.run_if) {   // one CTA per tile
    gemm_dmma_tile<C>(p, tiles_m, tiles_n, blockIdx.x, smem);
    return;
  }
  // the Ozaki guard's recomputation: a small persistent grid that does
  // nothing unless the guard set the flag (cheap when it did not)
  if (*reinterpret_cast<const volatile int *>(p.run_if) == 0) return;
  for (int bid = blockIdx.x; bid < tiles_m * tiles_n; bid += gridDim.x) {
    __syncthreads();   // the previous tile's shared-memory reads are done
    gemm_dmma_tile<C>(p, tiles_m, tiles_n, bid, smem);
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
  if (tm * tn > 0x7fffffffLL || p.splitk > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)(p.run_if ? std::min<int64_t>(tm * tn, 2 * 148) : tm * tn), 1,
            (unsigned)(p.splitk > 1 ? p.splitk : 1));
  kern<<<grid, C::NT, C::SMEM, s>>>(p, (int)tm, (int)tn);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// complex128 3M: CTA 64x64, BK 8, 8 warps of 32x16, 6 stages (A/B sweep in
// tools/gemm_lab.cu: BK 8 / 6 stages 44.0 TF/s vs BK 16 / 4 stages 41.6 on
// the chi=4096 GEMM4 shape)
template <bool AK, bool BK>
using Z3Cfg = Cfg<kCplx3M, 64, 64, 8, 32, 16, 6, AK, BK, 1>;
// complex128 4M: same tiling
template <bool AK, bool BK>
using Z4Cfg = Cfg<kCplx4M, 64, 64, 16, 32, 16, 4, AK, BK, 1>;
// float64: CTA 128x128, BK 16, 8 warps of 64x32, 3 stages
template <bool AK, bool BK, int VEC>
using DCfg = Cfg<kReal, 128, 128, 16, 64, 32, 3, AK, BK, VEC>;

template <template <bool, bool> class Z>
cudaError_t run_z(const GemmProblem &p, bool ak, bool bk, cudaStream_t s, int64_t *launches) {
  if (ak && bk) return run<Z<true, true>>(p, s, launches);
  if (ak && !bk) return run<Z<true, false>>(p, s, launches);
  if (!ak && bk) return run<Z<false, true>>(p, s, launches);
  return run<Z<false, false>>(p, s, launches);
}


}  // namespace

cudaError_t launch_gemm_f32(const GemmProblem &p, cudaStream_t s, int64_t *launches);

namespace {
// split-K reduction: C[m, n] = sum_{z ascending} partial[z][m][n] (fixed
// order -> deterministic); P = partial element, O = output element
template <typename P, typename O>
__global__ void __launch_bounds__(256) splitk_reduce(const P *__restrict__ part, O *__restrict__ C,
                                                     int64_t M, int64_t N, int64_t c_sm, int S,
                                                     const int64_t *c_row, const int64_t *c_col) {
  const int64_t MN = M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < MN; i += (int64_t)gridDim.x * blockDim.x) {
    P acc = part[i];
    for (int z = 1; z < S; z++) {
      const P v = part[(int64_t)z * MN + i];
      if constexpr (sizeof(P) == 16) {
        reinterpret_cast<double2 &>(acc).x += reinterpret_cast<const double2 &>(v).x;
        reinterpret_cast<double2 &>(acc).y += reinterpret_cast<const double2 &>(v).y;
      } else {
        reinterpret_cast<double &>(acc) += reinterpret_cast<const double &>(v);
      }
    }
    const int64_t m = i / N, n = i % N;
    const int64_t ci = c_row ? c_row[m] + c_col[n] : m * c_sm + n;
    if constexpr (sizeof(O) == sizeof(P)) {
      C[ci] = reinterpret_cast<const O &>(acc);
    } else if constexpr (sizeof(P) == 16) {
      const double2 a = reinterpret_cast<const double2 &>(acc);
      const float2 f = make_float2((float)a.x, (float)a.y);
      C[ci] = reinterpret_cast<const O &>(f);
    } else {
      const float f = (float)reinterpret_cast<const double &>(acc);
      C[ci] = reinterpret_cast<const O &>(f);
    }
  }
}
// Few outputs, many splits (thin / small GEMMs): a warp per output, lane l
// summing splits l, l + 32, ... in ascending order, then a fixed xor tree --
// deterministic, and the 148 SMs share the S reads of each output instead of
// one thread walking them
template <class P, class O>
__global__ void __launch_bounds__(256) splitk_reduce_w(const P *__restrict__ part, O *__restrict__ C,
                                                       int64_t M, int64_t N, int64_t c_sm, int S,
                                                       const int64_t *c_row, const int64_t *c_col) {
  const int64_t MN = M * N;
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < MN;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double ax = 0.0, ay = 0.0;
    for (int z = lane; z < S; z += 32) {
      const P v = part[(int64_t)z * MN + i];
      if constexpr (sizeof(P) == 16) {
        ax += reinterpret_cast<const double2 &>(v).x;
        ay += reinterpret_cast<const double2 &>(v).y;
      } else {
        ax += reinterpret_cast<const double &>(v);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      ax += __shfl_xor_sync(0xffffffffu, ax, o);
      if constexpr (sizeof(P) == 16) ay += __shfl_xor_sync(0xffffffffu, ay, o);
    }
    if (lane == 0) {
      const int64_t m = i / N, n = i % N;
      const int64_t ci = c_row ? c_row[m] + c_col[n] : m * c_sm + n;
      if constexpr (sizeof(P) == 16) {
        if constexpr (sizeof(O) == 16) {
          const double2 r = make_double2(ax, ay);
          C[ci] = reinterpret_cast<const O &>(r);
        } else {
          const float2 r = make_float2((float)ax, (float)ay);
          C[ci] = reinterpret_cast<const O &>(r);
        }
      } else {
        if constexpr (sizeof(O) == 8) {
          C[ci] = reinterpret_cast<const O &>(ax);
        } else {
          const float r = (float)ax;
          C[ci] = reinterpret_cast<const O &>(r);
        }
      }
    }
  }
}
}  // namespace

static cudaError_t launch_splitk_reduce(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  const int64_t MN = p.M * p.N;
  if (p.splitk >= 8 && MN < 148 * 256) {
    const unsigned blocks = (unsigned)std::min<int64_t>((MN + 7) / 8, 148 * 8);
    switch (p.dtype) {
      case TCI_C128:
        splitk_reduce_w<double2, double2><<<blocks, 256, 0, s>>>((const double2 *)p.partial, (double2 *)p.C, p.M, p.N, p.c_sm, p.splitk, p.c_row, p.c_col);
        break;
      case TCI_R64:
        splitk_reduce_w<double, double><<<blocks, 256, 0, s>>>((const double *)p.partial, (double *)p.C, p.M, p.N, p.c_sm, p.splitk, p.c_row, p.c_col);
        break;
      case TCI_C64:
        splitk_reduce_w<double2, float2><<<blocks, 256, 0, s>>>((const double2 *)p.partial, (float2 *)p.C, p.M, p.N, p.c_sm, p.splitk, p.c_row, p.c_col);
        break;
      case TCI_R32:
        splitk_reduce_w<double, float><<<blocks, 256, 0, s>>>((const double *)p.partial, (float *)p.C, p.M, p.N, p.c_sm, p.splitk, p.c_row, p.c_col);
        break;
    }
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  const unsigned blocks = (unsigned)std::min<int64_t>((MN + 255) / 256, 148 * 8);
  switch (p.dtype) {
    case TCI_C128:
      splitk_reduce<double2, double2><<<blocks, 256, 0, s>>>((const double2 *)p.partial, (double2 *)p.C, p.M, p.N, p.c_sm, p.splitk, p.c_row, p.c_col);
      break;
    case TCI_R64:
      splitk_reduce<double, double><<<blocks, 256, 0, s>>>((const double *)p.partial, (double *)p.C, p.M, p.N, p.c_sm, p.splitk, p.c_row, p.c_col);
      break;
    case TCI_C64:
      splitk_reduce<double2, float2><<<blocks, 256, 0, s>>>((const double2 *)p.partial, (float2 *)p.C, p.M, p.N, p.c_sm, p.splitk, p.c_row, p.c_col);
      break;
    case TCI_R32:
      splitk_reduce<double, float><<<blocks, 256, 0, s>>>((const double *)p.partial, (float *)p.C, p.M, p.N, p.c_sm, p.splitk, p.c_row, p.c_col);
      break;
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

void gemm_tile(tci_dtype_t dtype, int *bm, int *bn) {
  const bool big = dtype == TCI_R64 || dtype == TCI_R32;
  *bm = big ? 128 : 64;
  *bn = big ? 128 : 64;
}

static cudaError_t launch_gemm_main(const GemmProblem &p, cudaStream_t s, int64_t *launches);

cudaError_t launch_gemm(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  cudaError_t e = launch_gemm_main(p, s, launches);
  if (e != cudaSuccess || p.splitk <= 1 || p.M == 0 || p.N == 0) return e;
  return launch_splitk_reduce(p, s, launches);
}

bool tebd_fused_supported(const TebdProblem &t) {
  auto al16 = [](const void *x) { return ((uintptr_t)x % 16) == 0; };
  return t.d == 2 && t.a_b == 1 && t.b_c == 1 && al16(t.A) && al16(t.B) && t.a_a % 2 == 0 &&
         t.a_s % 2 == 0 && t.b_b % 2 == 0 && t.b_t % 2 == 0 && t.chi_b >= 1;
}

cudaError_t launch_tebd_fused(const TebdProblem &t, cudaStream_t s, int64_t *launches) {
  using TC = Cfg<kReal, 128, 128, 16, 64, 32, 3, true, false, 2, 1>;
  GemmProblem p{};
  p.dtype = TCI_R64;
  p.M = 2 * t.chi_a;
  p.N = 2 * t.chi_c;
  p.K = t.chi_b;
  p.A = t.A; p.a_sm = 0; p.a_sk = 1;
  p.B = t.B; p.b_sk = t.b_b; p.b_sn = 1;
  p.mode = 1;
  p.te_chi_a = t.chi_a; p.te_chi_c = t.chi_c;
  p.te_a_a = t.a_a; p.te_a_s = t.a_s; p.te_b_t = t.b_t;
  p.te_U = t.U;
  p.te_u[0] = t.u_p; p.te_u[1] = t.u_q; p.te_u[2] = t.u_s; p.te_u[3] = t.u_t;
  p.te_T = t.T;
  p.te_t[0] = t.t_a; p.te_t[1] = t.t_p; p.te_t[2] = t.t_q; p.te_t[3] = t.t_c;
  return run<TC>(p, s, launches);   // tiles: (chi_a / 64) x (chi_c / 64)
}

cudaError_t launch_gemm_dmma_if(const GemmProblem &p, const int *run_if, cudaStream_t s, int64_t *launches) {
  GemmProblem q = p;
  q.zalgo = kZ3M;
  q.run_if = run_if;
  q.npeer = 0;
  q.rows_done = nullptr;
  q.rows_needed = nullptr;
  return launch_gemm_main(q, s, launches);
}

static cudaError_t launch_gemm_main(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  if (p.M == 0 || p.N == 0) return cudaSuccess;
  // one of M, N, K tiny: HBM-bound, no tensor-core tile (gemm_thin.cu)
  if (gemm_thin_applies(p)) return launch_gemm_thin(p, s, launches);
  if (p.dtype == TCI_R32 || p.dtype == TCI_C64) {
    // float32 / complex64 on the INT8 tensor cores (Ozaki-II, t >= 24: R34)
    if (p.zalgo == kZOzaki && p.splitk <= 1 && p.mode == 0 && !p.c_row)
      return p.dtype == TCI_C64 ? launch_ozaki_zgemm(p, p.oz_ws, p.oz_ws_bytes, s, launches)
                                : launch_ozaki_dgemm(p, p.oz_ws, p.oz_ws_bytes, s, launches);
    return launch_gemm_f32(p, s, launches);
  }
  // The planner canonicalises strides (contract.cpp): a_sk == 1 selects the
  // K-contiguous loader, otherwise a_sm == 1; same for B.
  const bool ak = (p.a_sk == 1), bk = (p.b_sk == 1);
  if (p.dtype == TCI_C128) {
    if (p.zalgo == kZOzaki && p.splitk <= 1) return launch_ozaki_zgemm(p, p.oz_ws, p.oz_ws_bytes, s, launches);
    return p.zalgo == kZ4M ? run_z<Z4Cfg>(p, ak, bk, s, launches) : run_z<Z3Cfg>(p, ak, bk, s, launches);
  }
  // float64 on the INT8 tensor cores (real Ozaki-II) when the caller chose it
  if (p.zalgo == kZOzaki && p.splitk <= 1 && p.mode == 0 && !p.c_row)
    return launch_ozaki_dgemm(p, p.oz_ws, p.oz_ws_bytes, s, launches);
  // float64: 16-byte chunks need 16-byte aligned rows
  const int64_t lda = ak ? p.a_sm : p.a_sk, ldb = bk ? p.b_sn : p.b_sk;
  const bool aligned = ((uintptr_t)p.A % 16 == 0) && ((uintptr_t)p.B % 16 == 0) &&
                       (lda % 2 == 0 || (ak ? p.M : p.K) == 1) &&
                       (ldb % 2 == 0 || (bk ? p.N : p.K) == 1);
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
