// ozaki.cu -- complex128 / float64 GEMM on the INT8 tensor cores (tcgen05
// kind::i8) by the Ozaki-II integer-modular scheme (DESIGN.md
// §12, reading R26):
//
//   0. balance: per contraction index k an exact power of two 2^{s_k} moves
//      between A's column k and B's row k (A diag(2^s) diag(2^-s) B = AB),
//      s_k = floor((KB_k - KA_k)/2) from the per-k maxima, so entries that
//      multiply each other sit on a common scale;
//   1. scale: for every row m of A (re and im) pick E_m with |A'(m,k)| < 2^E_m
//      and round A'(m,k) 2^(t - E_m) to a t-bit integer (exact in fp64);
//      likewise the columns of B';
//   2. the integer complex product C' = A'B' is computed EXACTLY from its
//      residues modulo n coprime moduli m_l <= 255 (prod m_l > 4 max|C'|):
//      with the 3M split (exact in integer arithmetic)
//        P = A'r B'r,  Q = A'i B'i,  S = (A'r + A'i)(B'r + B'i),
//        C'r = P - Q,  C'i = S - P - Q,
//      every residue operand is an int8 in [-127, 127] and all 3n INT8 GEMMs
//      (int32 accumulation, exact for K <= 131072) run in ONE launch of the
//      hand-written tcgen05 kernel of i8gemm.cu, which leaves each product
//      reduced mod m_l as a byte;
//   3. CRT: C' = sum_l c_l w_l mod M (w_l the CRT weights, M = prod m_l) in
//      exact chunked fp64 integer arithmetic, converted to fp64 and scaled
//      back by 2^-(2t - E_m - E_n);
//   4. guard: the expected squared truncation error (independent roundings,
//      R26) against ||C||_F on the device; above the tolerance the product is
//      recomputed on DMMA by a launch gated on a device flag.
//
// The only roundings are step 1's truncation (|delta| <= 2^(E_m - t - 1) per
// component) and the final conversion. t and n are chosen from K:
// 2t + 3 + log2 K <= log2 M. Rows are processed in chunks so the residue
// planes and byte outputs fit a bounded workspace.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

constexpr int kMaxMod = 15;
// bit budget of float32 / complex64 sources (R34): operand entries keep 24
// bits relative to their line maximum -- every entry within 2^0 of it is
// exact (a float32 mantissa), smaller ones round as fp32 arithmetic would
constexpr int kOzTminF32 = kOzakiTminF32;
constexpr int kModuli[kMaxMod] = {255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
__constant__ int c_moduli[kMaxMod] = {255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};

// Gaussian moduli of the complex path (R33): odd, pairwise
// coprime, every prime factor = 1 mod 4 (221 = 13 17, 205 = 5 41), so -1 has
// a square root j_l mod m_l (kGRoots: the balanced one, j^2 = -1 mod m) and
// a + ib -> (a + j b, a - j b) mod m is a ring homomorphism Z[i] -> Z_m x Z_m:
// a complex product mod m costs two real products instead of three (3M).
constexpr int kMaxGMod = 16;
constexpr int kGModuli[kMaxGMod] = {241, 233, 229, 221, 205, 197, 193, 181, 173, 157, 149, 137, 113, 109, 101, 97};
constexpr int kGRoots[kMaxGMod] = {64, 89, 107, 21, 32, 14, 81, 19, 80, 28, 44, 37, 15, 33, 10, 22};
__constant__ int c_gmod[kMaxGMod] = {241, 233, 229, 221, 205, 197, 193, 181, 173, 157, 149, 137, 113, 109, 101, 97};
__constant__ int c_groot[kMaxGMod] = {64, 89, 107, 21, 32, 14, 81, 19, 80, 28, 44, 37, 15, 33, 10, 22};
// negated moduli and roots (so every integer step of gauss_planes is one IMAD)
__constant__ int c_gnmod[kMaxGMod] = {-241, -233, -229, -221, -205, -197, -193, -181, -173, -157, -149, -137, -113, -109, -101, -97};
__constant__ int c_gnroot[kMaxGMod] = {-64, -89, -107, -21, -32, -14, -81, -19, -80, -28, -44, -37, -15, -33, -10, -22};
__constant__ double c_grootd[kMaxGMod] = {64, 89, 107, 21, 32, 14, 81, 19, 80, 28, 44, 37, 15, 33, 10, 22};
__constant__ double c_gminv[kMaxGMod] = {1.0 / 241, 1.0 / 233, 1.0 / 229, 1.0 / 221, 1.0 / 205, 1.0 / 197,
                                         1.0 / 193, 1.0 / 181, 1.0 / 173, 1.0 / 157, 1.0 / 149, 1.0 / 137,
                                         1.0 / 113, 1.0 / 109, 1.0 / 101, 1.0 / 97};
__constant__ float c_gminvf[kMaxGMod] = {1.0f / 241, 1.0f / 233, 1.0f / 229, 1.0f / 221, 1.0f / 205, 1.0f / 197,
                                         1.0f / 193, 1.0f / 181, 1.0f / 173, 1.0f / 157, 1.0f / 149, 1.0f / 137,
                                         1.0f / 113, 1.0f / 109, 1.0f / 101, 1.0f / 97};

// ---------------------------------------------------------------------------
// Small helpers: exact powers of two, exponent / mantissa split
// ---------------------------------------------------------------------------
__device__ __forceinline__ double pow2i(int h) {   // 2^h, h <= 1023; 0 below the normal range
  return h < -1022 ? 0.0 : __hiloint2double((h + 1023) << 20, 0);
}
__device__ __forceinline__ double pow4i(int d) { return d < -511 ? 0.0 : pow2i(2 * d); }   // 4^d, d <= 0

// the two exact power-of-two factors a * b = 2^sc used by scaled_magic
__device__ __forceinline__ void scale_pair(int sc, double &a, double &b) {
  const int h1 = sc >> 1, h2 = sc - h1;
  if (h1 >= -1022 && h2 <= 1023) {
    a = __hiloint2double((h1 + 1023) << 20, 0);
    b = __hiloint2double((h2 + 1023) << 20, 0);
  } else {
    a = ldexp(1.0, h1);
    b = ldexp(1.0, h2);
  }
}

// ---------------------------------------------------------------------------
// step 0 (K-balancing, R26): for every contraction index k the
// exponent KX_k with |x| < 2^KX_k over all lines of one operand (re and im)
// and the normalised sum of squares S_k = sum |x|^2 4^-KX_k. An online
// (exponent, sum) pair: a larger exponent rescales the sum by a power of 4;
// pairs merge in a fixed order (deterministic).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void es_add(int &em, double &s, double x) {
  if (x == 0.0) return;
  int e;
  const double f = frexp(x, &e);
  if (e > em) {
    s = em == -100000 ? 0.0 : s * pow4i(em - e);
    em = e;
  }
  s = fma(f * f, pow4i(e - em), s);
}
__device__ __forceinline__ void es_merge(int &em, double &s, int e2, double s2) {
  if (e2 == -100000) return;
  if (e2 > em) {
    s = em == -100000 ? 0.0 : s * pow4i(em - e2);
    em = e2;
  }
  s = fma(s2, pow4i(e2 - em), s);
}
__device__ __forceinline__ void es_add(int &em, double &s, double2 x) {
  es_add(em, s, x.x);
  es_add(em, s, x.y);
}
// float32 sources (exact widening)
__device__ __forceinline__ void es_add(int &em, double &s, float x) { es_add(em, s, (double)x); }
__device__ __forceinline__ void es_add(int &em, double &s, float2 x) {
  es_add(em, s, (double)x.x);
  es_add(em, s, (double)x.y);
}

// per-k statistics when the lines are contiguous (s_l == 1): one warp per k,
// lanes walk the lines, fixed xor-tree merge
template <class T>
__global__ void __launch_bounds__(256) kstats_lines(const T *X, int64_t K, int64_t L, int64_t s_k, int *KE,
                                                    double *KS) {
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= K) return;
  int em = -100000;
  double s = 0.0;
  const T *p = X + k * s_k;
  for (int64_t l = lane; l < L; l += 32) es_add(em, s, __ldg(p + l));
  for (int o = 16; o; o >>= 1) {
    const int e2 = __shfl_xor_sync(0xffffffffu, em, o);
    const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
    // both lanes of a pair must end with the same value: merge in lane order
    if (lane & o) {
      int ea = e2;
      double sa = s2;
      es_merge(ea, sa, em, s);
      em = ea;
      s = sa;
    } else {
      es_merge(em, s, e2, s2);
    }
  }
  if (lane == 0) {
    KE[k] = em;
    KS[k] = s;
  }
}

// per-k statistics when k is contiguous: thread per k (coalesced), blockIdx.y
// takes a chunk of lines; partial pairs go to slots [chunk][k]
template <class T>
__global__ void __launch_bounds__(256) kstats_cols(const T *X, int64_t K, int64_t L, int64_t s_l, int64_t chunk,
                                                   int *SE, double *SS) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int64_t l0 = blockIdx.y * chunk, l1 = min(L, l0 + chunk);
  int em = -100000;
  double s = 0.0;
  const T *p = X + k;
  int64_t l = l0;
  for (; l + 4 <= l1; l += 4) {
    const T v0 = __ldg(p + l * s_l), v1 = __ldg(p + (l + 1) * s_l);
    const T v2 = __ldg(p + (l + 2) * s_l), v3 = __ldg(p + (l + 3) * s_l);
    es_add(em, s, v0);
    es_add(em, s, v1);
    es_add(em, s, v2);
    es_add(em, s, v3);
  }
  for (; l < l1; l++) es_add(em, s, __ldg(p + l * s_l));
  SE[blockIdx.y * K + k] = em;
  SS[blockIdx.y * K + k] = s;
}

// ---- fused pass (round 2): the per-k statistics AND the unbalanced per-line
// exponents E (max over k of the frexp exponents, re and im) from ONE read of
// the operand; when the K-balancing then turns out inactive (the common case)
// E is final and the separate line_exponent pass is skipped (it runs gated on
// the device flag otherwise). Same (exponent, sum) arithmetic and merge orders
// as kstats_lines / kstats_cols: the statistics are bitwise the same.
__device__ __forceinline__ int es_add_e(int &em, double &s, double x) {   // returns x's exponent
  if (x == 0.0) return -100000;
  int e;
  const double f = frexp(x, &e);
  if (e > em) {
    s = em == -100000 ? 0.0 : s * pow4i(em - e);
    em = e;
  }
  s = fma(f * f, pow4i(e - em), s);
  return e;
}
__device__ __forceinline__ int es_add_e(int &em, double &s, double2 x) {
  const int a = es_add_e(em, s, x.x), b = es_add_e(em, s, x.y);
  return max(a, b);
}
__device__ __forceinline__ int es_add_e(int &em, double &s, float x) { return es_add_e(em, s, (double)x); }
__device__ __forceinline__ int es_add_e(int &em, double &s, float2 x) {
  const int a = es_add_e(em, s, (double)x.x), b = es_add_e(em, s, (double)x.y);
  return max(a, b);
}

// K-contiguous lines (s_k == 1): thread per k (coalesced), the block's chunk
// of lines in order; line maxima by a warp max + shared atomicMax, then one
// global atomicMax per line and block (max is order-independent)
template <class T>
__global__ void __launch_bounds__(256) kstats_cols_lx(const T *X, int64_t K, int64_t L, int64_t s_l, int64_t chunk,
                                                      int *SE, double *SS, int *E) {
  extern __shared__ int sE[];
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t l0 = blockIdx.y * chunk, l1 = min(L, l0 + chunk);
  for (int64_t i = threadIdx.x; i < l1 - l0; i += blockDim.x) sE[i] = -100000;
  __syncthreads();
  const bool kin = k < K;
  int em = -100000;
  double s = 0.0;
  const T *p = X + (kin ? k : 0);
#pragma unroll 4
  for (int64_t l = l0; l < l1; l++) {
    int ex = -100000;
    if (kin) ex = es_add_e(em, s, __ldg(p + l * s_l));
    const int wm = __reduce_max_sync(0xffffffffu, ex);
    if ((threadIdx.x & 31) == 0 && wm > -100000) atomicMax(&sE[l - l0], wm);
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < l1 - l0; i += blockDim.x)
    if (sE[i] > -100000) atomicMax(E + l0 + i, sE[i]);
  if (kin) {
    SE[blockIdx.y * K + k] = em;
    SS[blockIdx.y * K + k] = s;
  }
}

// line-contiguous lines (s_l == 1): warp per k as kstats_lines (lanes walk
// the chunk's lines, coalesced; the same xor-tree merge), 4 k per warp and
// 32 per block; line maxima by shared atomicMax over the block's 32 k, then
// one global atomicMax per line and block
template <class T>
__global__ void __launch_bounds__(256) kstats_lines_lx(const T *X, int64_t K, int64_t L, int64_t s_k, int64_t chunk,
                                                       int *SE, double *SS, int *E) {
  extern __shared__ int sE[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t l0 = blockIdx.y * chunk, l1 = min(L, l0 + chunk);
  for (int64_t i = threadIdx.x; i < l1 - l0; i += blockDim.x) sE[i] = -100000;
  __syncthreads();
  // the warp's 4 k per line in registers: one shared atomicMax per line and warp
  const int64_t kb = blockIdx.x * 32 + warp * 4;
  int em[4];
  double sv[4];
#pragma unroll
  for (int kk = 0; kk < 4; kk++) {
    em[kk] = -100000;
    sv[kk] = 0.0;
  }
  for (int64_t l = l0 + lane; l < l1; l += 32) {
    int lmax = -100000;
#pragma unroll
    for (int kk = 0; kk < 4; kk++)
      if (kb + kk < K) lmax = max(lmax, es_add_e(em[kk], sv[kk], __ldg(X + (kb + kk) * s_k + l)));
    if (lmax > -100000) atomicMax(&sE[l - l0], lmax);
  }
#pragma unroll
  for (int kk = 0; kk < 4; kk++) {
    int e = em[kk];
    double sk = sv[kk];
    for (int o = 16; o; o >>= 1) {
      const int e2 = __shfl_xor_sync(0xffffffffu, e, o);
      const double s2 = __shfl_xor_sync(0xffffffffu, sk, o);
      if (lane & o) {
        int ea = e2;
        double sa = s2;
        es_merge(ea, sa, e, sk);
        e = ea;
        sk = sa;
      } else {
        es_merge(e, sk, e2, s2);
      }
    }
    if (lane == 0 && kb + kk < K) {
      SE[blockIdx.y * K + kb + kk] = e;
      SS[blockIdx.y * K + kb + kk] = sk;
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < l1 - l0; i += blockDim.x)
    if (sE[i] > -100000) atomicMax(E + l0 + i, sE[i]);
}

__global__ void __launch_bounds__(256) kstats_merge(const int *SE, const double *SS, int nch, int64_t K, int *KE,
                                                    double *KS) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  int em = -100000;
  double s = 0.0;
  for (int c = 0; c < nch; c++) es_merge(em, s, SE[c * K + k], SS[c * K + k]);
  KE[k] = em;
  KS[k] = s;
}

// s_k = floor((KB_k - KA_k) / 2): after A(:,k) 2^s_k and B(k,:) 2^-s_k both
// maxima are within a factor 2 of their geometric mean (0 where either line
// is all zero). A spread max_k s_k - min_k s_k <= 2 changes the truncation
// error by at most ~4x: then no balancing (s = 0; bal = 0 keeps the per-line
// fast path and the results bitwise those of the plain scheme).
// Single block. SK has Kp entries (zero beyond K).
__global__ void __launch_bounds__(1024) balance_prep(const int *KA, const int *KB, int64_t K, int64_t Kp, int enable,
                                                     int *SK, int *bal) {
  __shared__ int smin[32], smax[32];
  __shared__ int use;
  int lo = INT32_MAX, hi = INT32_MIN;
  auto sval = [&](int64_t k) {
    const int a = KA[k], b = KB[k];
    if (a == -100000 || b == -100000) return 0;
    return max(-500, min(500, (b - a) >> 1));   // arithmetic shift = floor
  };
  if (enable)
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
      if (KA[k] == -100000 || KB[k] == -100000) continue;
      const int v = sval(k);
      lo = min(lo, v);
      hi = max(hi, v);
    }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = lo;
    smax[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = INT32_MAX, b = INT32_MIN;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
      a = min(a, smin[w]);
      b = max(b, smax[w]);
    }
    use = enable && a <= b && b - a > 2;
    *bal = use;
  }
  __syncthreads();
  for (int64_t k = threadIdx.x; k < Kp; k += blockDim.x) SK[k] = (use && k < K) ? sval(k) : 0;
}

// ---------------------------------------------------------------------------
// step 1a: per-row (A) / per-column (B) exponent E with |x 2^(sgn s_k)| < 2^E
// for every entry (re and im) of that row/column; E = -100000 for an
// all-zero line. SK / bal: the K-balancing (applied when *bal != 0).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int exp_of(double x) {
  if (x == 0.0) return -100000;
  int e;
  frexp(x, &e);   // |x| = f 2^e, 0.5 <= f < 1  ->  |x| < 2^e
  return e;
}
__device__ __forceinline__ int exp_of(double2 v) { return max(exp_of(v.x), exp_of(v.y)); }
__device__ __forceinline__ int exp_of(float v) { return exp_of((double)v); }
__device__ __forceinline__ int exp_of(float2 v) { return max(exp_of((double)v.x), exp_of((double)v.y)); }
__device__ __forceinline__ int exp_of_shift(float2 v, int s) {
  const int e = exp_of(v);
  return e == -100000 ? e : e + s;
}
__device__ __forceinline__ int exp_of_shift(float v, int s) {
  const int e = exp_of(v);
  return e == -100000 ? e : e + s;
}
// operand loads widened to double (float32 sources: exact)
__device__ __forceinline__ double2 ld_c(const double2 *p) { return __ldg(p); }
__device__ __forceinline__ double2 ld_c(const float2 *p) {
  const float2 v = __ldg(p);
  return make_double2(v.x, v.y);
}
__device__ __forceinline__ double ld_r(const double *p) { return __ldg(p); }
__device__ __forceinline__ double ld_r(const float *p) { return (double)__ldg(p); }
// result stores (streaming); float32 results are rounded once
__device__ __forceinline__ void st_c(double2 *p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_c(float2 *p, double2 v) { __stcs(p, make_float2((float)v.x, (float)v.y)); }
__device__ __forceinline__ void st_r(double *p, double v) { *p = v; }
__device__ __forceinline__ void st_r(float *p, double v) { *p = (float)v; }
__device__ __forceinline__ int exp_of_shift(double2 v, int s) {
  const int e = exp_of(v);
  return e == -100000 ? e : e + s;
}
__device__ __forceinline__ int exp_of_shift(double v, int s) {
  const int e = exp_of(v);
  return e == -100000 ? e : e + s;
}

// line l (= m for A, n for B) of extent K; element (l, k) at base + l*s_l + k*s_k.
// K-contiguous lines: one warp per line. Line-contiguous (s_l == 1):
// blockIdx.y splits K into chunks, consecutive threads take consecutive lines
// (coalesced) and combine with atomicMax (max is order-independent:
// deterministic). E must be pre-set to -100000 in that mode.
template <class T>
__global__ void __launch_bounds__(256) line_exponent(const T *base, int64_t nlines, int64_t K, int64_t s_l,
                                                     int64_t s_k, int *E, const int *SK, int sgn,
                                                     const int *bal, int only_if_bal = 0) {
  const bool b = SK && *bal;
  if (only_if_bal && !b) return;   // the fused stats pass already left the unbalanced E
  if (s_k == 1) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= nlines) return;
    int e = -100000;
    const T *p = base + warp * s_l;
    if (b) {
      for (int64_t k = lane; k < K; k += 32) e = max(e, exp_of_shift(p[k], sgn * SK[k]));
    } else {
      for (int64_t k = lane; k < K; k += 32) e = max(e, exp_of(p[k]));
    }
    for (int o = 16; o; o >>= 1) e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
    if (lane == 0) E[warp] = e;
  } else {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= nlines) return;
    const int64_t kc = (K + gridDim.y - 1) / gridDim.y, k0 = blockIdx.y * kc;
    const int64_t k1 = min(K, k0 + kc);
    int e = -100000;
    const T *p = base + l * s_l;
    if (b) {
      for (int64_t k = k0; k < k1; k++) e = max(e, exp_of_shift(p[k * s_k], sgn * SK[k]));
    } else {
      for (int64_t k = k0; k < k1; k++) e = max(e, exp_of(p[k * s_k]));
    }
    atomicMax(E + l, e);
  }
}

__global__ void fill_int(int *p, int64_t n, int v, const int *only_if = nullptr) {
  if (only_if && !*only_if) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// max of E[0..n) into *out (single block; the guard's normalisation of the
// CRT's row sums)
__global__ void __launch_bounds__(1024) exp_max(const int *E, int64_t n, int *out) {
  __shared__ int sm[32];
  int v = -100000;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v = max(v, E[i]);
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) v = max(v, sm[w]);
    *out = max(v, sm[0]);
  }
}

// 1/m_l rounded to double (IEEE division, evaluated at compile time)
__constant__ double c_minv[kMaxMod] = {1.0 / 255, 1.0 / 253, 1.0 / 251, 1.0 / 247, 1.0 / 241, 1.0 / 239, 1.0 / 233, 1.0 / 229, 1.0 / 227, 1.0 / 223, 1.0 / 217, 1.0 / 211, 1.0 / 199, 1.0 / 197, 1.0 / 193};

constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52: x + kMagic rounds x to an integer (|x| < 2^51)

// rint(v * 2^sc) + 1.5*2^52 with the scale split in two exact power-of-two
// factors (s2a * s2b = 2^sc; the first product is inexact only when it is
// subnormal, and then the result rounds to 0 either way): the integer
// x = rint(v 2^sc) sits in the low mantissa bits, so x = result - kMagic and
// the low word of the result is x mod 2^32. Bitwise equal to rint(ldexp(v, sc)).
__device__ __forceinline__ double scaled_magic(double v, double s2a, double s2b) {
  return fma(v * s2a, s2b, kMagic);
}

// balanced residue r of an integer-valued double |x| < 2^51 modulo odd m,
// r in [-(m-1)/2, (m-1)/2]: q = rint(x/m) is exact (x/m is never within
// 2^-9.6 of a half-integer for odd m) and sits in the low word of
// fma(x, 1/m, 1.5*2^52); r = x - q m holds exactly in 32-bit wrap-around
// arithmetic on the low words (|r| < 2^31): one DFMA + one IMAD per residue
__device__ __forceinline__ int bal_res(double x, int x_lo, double minv, int m) {
  return x_lo - __double2loint(fma(x, minv, kMagic)) * m;
}

// low bytes of four ints -> one word (3 PRMT)
__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return __byte_perm(__byte_perm((uint32_t)a, (uint32_t)b, 0x0040), __byte_perm((uint32_t)c, (uint32_t)d, 0x0040),
                     0x5410);
}

// Scaled integers of NV consecutive complex values: x[0] = re, x[1] = im,
// x[2] = re + im (exact, |.| < 2^49) and their low words
template <int NV>
struct ResVals {
  double x[3][NV];
  int lo[3][NV];
  __device__ __forceinline__ void set(int j, double mr, double mi) {   // mr, mi: scaled_magic outputs
    x[0][j] = mr - kMagic;
    x[1][j] = mi - kMagic;
    x[2][j] = x[0][j] + x[1][j];
    lo[0][j] = __double2loint(mr);
    lo[1][j] = __double2loint(mi);
    lo[2][j] = lo[0][j] + lo[1][j];
  }
};

// the three residue planes (re, im, re + im) of NV consecutive values for
// modulus l, packed 4 bytes per word
template <int NV>
__device__ __forceinline__ void residue_words(const ResVals<NV> &v, int l, uint32_t (&w)[3][NV / 4]) {
  const int mi = c_moduli[l];
  const double minv = c_minv[l];
#pragma unroll
  for (int c = 0; c < 3; c++)
#pragma unroll
    for (int q = 0; q < NV / 4; q++)
      w[c][q] = pack4(bal_res(v.x[c][q * 4 + 0], v.lo[c][q * 4 + 0], minv, mi),
                      bal_res(v.x[c][q * 4 + 1], v.lo[c][q * 4 + 1], minv, mi),
                      bal_res(v.x[c][q * 4 + 2], v.lo[c][q * 4 + 2], minv, mi),
                      bal_res(v.x[c][q * 4 + 3], v.lo[c][q * 4 + 3], minv, mi));
}

// balanced residue of a small integer |u| < 2^22 modulo odd m < 256: the
// quotient rint(u/m) sits in the low mantissa bits of fma(u, 1/m, 1.5 2^23)
// (|u/m - rint(u/m)| >= 1/(2m) > the fp32 error |u| 2^-24 / m)
__device__ __forceinline__ int small_bal(int u, float minvf, int m) {
  // (float)u without an I2F (XU pipe): u sits in the low mantissa bits of 1.5 2^23 + u
  const float uf = __int_as_float(0x4B400000 + u) - 12582912.0f;
  const float q = fmaf(uf, minvf, 12582912.0f);
  return u - (__float_as_int(q) - 0x4B400000) * m;
}

// the two Gaussian residue planes (a + j b, a - j b) mod m_l of NV
// consecutive values (x[0] = re, x[1] = im), balanced, packed 4 bytes per word
template <int NV>
__device__ __forceinline__ void residue_words_g(const ResVals<NV> &v, int l, uint32_t (&w)[2][NV / 4]) {
  const int mi = c_gmod[l], jr = c_groot[l];
  const double minv = c_gminv[l];
  const float minvf = c_gminvf[l];
  int u[NV], d[NV];
#pragma unroll
  for (int j = 0; j < NV; j++) {
    const int rr = bal_res(v.x[0][j], v.lo[0][j], minv, mi);
    const int ri = bal_res(v.x[1][j], v.lo[1][j], minv, mi);
    const int tj = jr * ri;   // |.| <= 120 * 120
    u[j] = small_bal(rr + tj, minvf, mi);
    d[j] = small_bal(rr - tj, minvf, mi);
  }
#pragma unroll
  for (int q = 0; q < NV / 4; q++) {
    w[0][q] = pack4(u[q * 4 + 0], u[q * 4 + 1], u[q * 4 + 2], u[q * 4 + 3]);
    w[1][q] = pack4(d[q * 4 + 0], d[q * 4 + 1], d[q * 4 + 2], d[q * 4 + 3]);
  }
}

// the residue planes of one modulus (3M: re, im, re + im; Gaussian: a + jb,
// a - jb) stored at dst + (l * PPM + c) * plane_stride, 8 bytes per plane
template <bool G, int NV>
__device__ __forceinline__ void store_planes(const ResVals<NV> &x, int l, int8_t *dst, int64_t plane_stride) {
  static_assert(NV == 8, "8 values per thread");
  if constexpr (G) {
    uint32_t w[2][NV / 4];
    residue_words_g<NV>(x, l, w);
#pragma unroll
    for (int comp = 0; comp < 2; comp++)
      *reinterpret_cast<uint2 *>(dst + (int64_t)(l * 2 + comp) * plane_stride) = make_uint2(w[comp][0], w[comp][1]);
  } else {
    uint32_t w[3][NV / 4];
    residue_words<NV>(x, l, w);
#pragma unroll
    for (int comp = 0; comp < 3; comp++)
      *reinterpret_cast<uint2 *>(dst + (int64_t)(l * 3 + comp) * plane_stride) = make_uint2(w[comp][0], w[comp][1]);
  }
}

// scale factors 2^sc = s2a * s2b of one line (E > -100000)
__device__ __forceinline__ void line_scale(int t, int E, double &s2a, double &s2b) {
  const int sc = t - E, h1 = sc / 2;
  s2a = ldexp(1.0, h1);
  s2b = ldexp(1.0, sc - h1);
}

// ---------------------------------------------------------------------------
// step 1b + 2a: residue planes. out[(l*3 + comp)][line][kp] int8, K-major,
// comp 0 = re, 1 = im, 2 = re + im; zero for k >= K or line >= nlines.
// Each thread produces 8 consecutive k of one line for all planes. With the
// K-balancing active the scale of entry (line, k) is 2^(t - E_line + sgn s_k).
// ---------------------------------------------------------------------------
struct ResArgs {
  const void *base;         // double2 (complex) / double (real)
  int64_t nlines, K, Kp, s_l, s_k;
  int64_t line0;            // first line of the chunk (global index)
  int64_t lines_out;        // rows in the output planes (chunk, padded)
  const int *E;             // exponents (global line index)
  int t;                    // bit budget
  int nmod;
  int8_t *out;
  int64_t plane_stride;     // lines_out * Kp
  const int *SK;            // K-balancing exponents (Kp entries) or null
  const int *bal;           // device flag: balancing active
  int sgn;                  // +1 for A, -1 for B
  // Gaussian planes (R33): the moduli in groups [gfirst[g], gfirst[g+1]) whose
  // products P_g < 2^44 (odd) reduce each integer once per group
  double gP[3], gPinv[3];
  int gPlo[3], gfirst[4];
};

// The two Gaussian planes of every modulus for 8 values of one line (R33).
// Per group: x = q P + r_P exactly (q = rint(x / P) from one DFMA, r_P by a
// second, its low word by an IMAD on the low words), so every modulus of the
// group works on |r_P| < 2^43 instead of |x| < 2^49: x_u = r_P(re) + j r_P(im)
// is an exact double (|x_u| < 2^50) whose balanced residue needs one DFMA
// (the quotient) and one IMAD on the low words (lo(x_u) = lo(r_re) + j lo(r_im)).
// 2 DFMA + 5 integer ops per modulus and value instead of 2 full reductions of
// re and im plus two small ones (the kernel was instruction-issue bound).
template <int NV>
__device__ __forceinline__ void gauss_planes(const ResVals<NV> &v, const ResArgs &a, int8_t *dst) {
  static_assert(NV == 4 || NV == 8, "4 or 8 values per thread");
  const int64_t ps2 = 2 * a.plane_stride;
#pragma unroll 1
  for (int g = 0; g < 3; g++) {
    const int l0 = a.gfirst[g], l1 = min(a.gfirst[g + 1], a.nmod);
    if (l0 >= l1) break;
    const double P = a.gP[g], Pinv = a.gPinv[g];
    const int nPlo = -a.gPlo[g];
    double rp[NV], ip[NV];
    int lr[NV], li[NV];
#pragma unroll
    for (int j = 0; j < NV; j++) {
      const double mr = fma(v.x[0][j], Pinv, kMagic), mi = fma(v.x[1][j], Pinv, kMagic);
      rp[j] = fma(kMagic - mr, P, v.x[0][j]);   // x - q P, q = mr - kMagic (exact)
      ip[j] = fma(kMagic - mi, P, v.x[1][j]);
      lr[j] = __double2loint(mr) * nPlo + v.lo[0][j];
      li[j] = __double2loint(mi) * nPlo + v.lo[1][j];
    }
    int8_t *du = dst + l0 * ps2;
#pragma unroll 1
    for (int l = l0; l < l1; l++, du += ps2) {
      // every integer step one IMAD: lo(x_u) = li j + lr, r = q (-m) + lo(x_u)
      const int nm = c_gnmod[l], jr = c_groot[l], njr = c_gnroot[l];
      const double minv = c_gminv[l], jd = c_grootd[l];
      int u[NV], d[NV];
#pragma unroll
      for (int j = 0; j < NV; j++) {
        const double xu = fma(jd, ip[j], rp[j]), xd = fma(-jd, ip[j], rp[j]);
        u[j] = __double2loint(fma(xu, minv, kMagic)) * nm + (li[j] * jr + lr[j]);
        d[j] = __double2loint(fma(xd, minv, kMagic)) * nm + (li[j] * njr + lr[j]);
      }
      if constexpr (NV == 8) {
        *reinterpret_cast<uint2 *>(du) = make_uint2(pack4(u[0], u[1], u[2], u[3]), pack4(u[4], u[5], u[6], u[7]));
        *reinterpret_cast<uint2 *>(du + a.plane_stride) =
            make_uint2(pack4(d[0], d[1], d[2], d[3]), pack4(d[4], d[5], d[6], d[7]));
      } else {
        *reinterpret_cast<uint32_t *>(du) = pack4(u[0], u[1], u[2], u[3]);
        *reinterpret_cast<uint32_t *>(du + a.plane_stride) = pack4(d[0], d[1], d[2], d[3]);
      }
    }
  }
}

// the same with the moduli count known at compile time (15 or 16: the
// float64-source complex GEMMs): every loop unrolled, so the per-modulus
// constants are immediate constant-bank operands instead of indexed LDCs and
// the store addresses are constant offsets (groups 0-4, 5-9, 10-15 as in
// res_args)
template <int NV, int NMOD>
__device__ __forceinline__ void gauss_planes_ct(const ResVals<NV> &v, const ResArgs &a, int8_t *dst) {
  const int64_t ps = a.plane_stride;
#pragma unroll
  for (int g = 0; g < 3; g++) {
    const int l0 = 5 * g, l1 = g == 2 ? NMOD : 5 * (g + 1);
    const double P = a.gP[g], Pinv = a.gPinv[g];
    const int nPlo = -a.gPlo[g];
    double rp[NV], ip[NV];
    int lr[NV], li[NV];
#pragma unroll
    for (int j = 0; j < NV; j++) {
      const double mr = fma(v.x[0][j], Pinv, kMagic), mi = fma(v.x[1][j], Pinv, kMagic);
      rp[j] = fma(kMagic - mr, P, v.x[0][j]);
      ip[j] = fma(kMagic - mi, P, v.x[1][j]);
      lr[j] = __double2loint(mr) * nPlo + v.lo[0][j];
      li[j] = __double2loint(mi) * nPlo + v.lo[1][j];
    }
#pragma unroll
    for (int l = l0; l < l1; l++) {
      const int nm = c_gnmod[l], jr = c_groot[l], njr = c_gnroot[l];
      const double minv = c_gminv[l], jd = c_grootd[l];
      int u[NV], d[NV];
#pragma unroll
      for (int j = 0; j < NV; j++) {
        const double xu = fma(jd, ip[j], rp[j]), xd = fma(-jd, ip[j], rp[j]);
        u[j] = __double2loint(fma(xu, minv, kMagic)) * nm + (li[j] * jr + lr[j]);
        d[j] = __double2loint(fma(xd, minv, kMagic)) * nm + (li[j] * njr + lr[j]);
      }
      int8_t *du = dst + (int64_t)(2 * l) * ps;
      if constexpr (NV == 8) {
        *reinterpret_cast<uint2 *>(du) = make_uint2(pack4(u[0], u[1], u[2], u[3]), pack4(u[4], u[5], u[6], u[7]));
        *reinterpret_cast<uint2 *>(du + ps) = make_uint2(pack4(d[0], d[1], d[2], d[3]), pack4(d[4], d[5], d[6], d[7]));
      } else {
        *reinterpret_cast<uint32_t *>(du) = pack4(u[0], u[1], u[2], u[3]);
        *reinterpret_cast<uint32_t *>(du + ps) = pack4(d[0], d[1], d[2], d[3]);
      }
    }
  }
}

template <int NV>
__device__ __forceinline__ void gauss_planes_any(const ResVals<NV> &v, const ResArgs &a, int8_t *dst) {
  if (a.nmod == 15)
    gauss_planes_ct<NV, 15>(v, a, dst);
  else if (a.nmod == 16)
    gauss_planes_ct<NV, 16>(v, a, dst);
  else
    gauss_planes<NV>(v, a, dst);
}

// per-element scale factors of 8 consecutive k (SK has Kp >= k0 + 8 entries)// per-element scale factors of 8 consecutive k (SK has Kp >= k0 + 8 entries)
template <int NV = 8>
__device__ __forceinline__ void elem_scales(const ResArgs &a, int E, int64_t k0, double (&fa)[NV], double (&fb)[NV]) {
#pragma unroll
  for (int h = 0; h < NV / 4; h++) {
    const int4 q = *reinterpret_cast<const int4 *>(a.SK + k0 + 4 * h);
    const int s[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; j++) scale_pair(a.t - E + a.sgn * s[j], fa[4 * h + j], fb[4 * h + j]);
  }
}

template <bool G, class TS>
__global__ void __launch_bounds__(256, G ? 3 : 2) residues(const __grid_constant__ ResArgs a) {
  // Gaussian: 4 values per thread (more warps in flight: the kernel waits on
  // its loads), 4-byte stores per plane (a warp still writes 128 contiguous B)
  constexpr int NV = G ? 4 : 8;
  const int64_t kgroups = a.Kp / NV;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= a.lines_out * kgroups) return;
  // K-contiguous source: consecutive threads walk k (coalesced reads and writes)
  const int64_t row = gid / kgroups;
  const int64_t k0 = (gid % kgroups) * NV;
  const int64_t line = a.line0 + row;
  ResVals<NV> x;
  if (line < a.nlines && a.E[line] > -100000) {
    const TS *p = static_cast<const TS *>(a.base) + line * a.s_l;
    double2 v[NV];
#pragma unroll
    for (int j = 0; j < NV; j++) v[j] = k0 + j < a.K ? ld_c(p + (k0 + j) * a.s_k) : make_double2(0.0, 0.0);
    if (a.SK && *a.bal) {
      double fa[NV], fb[NV];
      elem_scales<NV>(a, a.E[line], k0, fa, fb);
#pragma unroll
      for (int j = 0; j < NV; j++) x.set(j, scaled_magic(v[j].x, fa[j], fb[j]), scaled_magic(v[j].y, fa[j], fb[j]));
    } else {
      const int sc = a.t - a.E[line];
      if (sc >= -1022 && sc <= 1023) {   // 2^sc normal: one DFMA per component (v 2^sc exact)
        const double f = pow2i(sc);
#pragma unroll
        for (int j = 0; j < NV; j++) x.set(j, fma(v[j].x, f, kMagic), fma(v[j].y, f, kMagic));
      } else {
        double s2a, s2b;
        line_scale(a.t, a.E[line], s2a, s2b);
#pragma unroll
        for (int j = 0; j < NV; j++) x.set(j, scaled_magic(v[j].x, s2a, s2b), scaled_magic(v[j].y, s2a, s2b));
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NV; j++) x.set(j, kMagic, kMagic);
  }
  int8_t *dst = a.out + row * a.Kp + k0;
  if constexpr (G)
    gauss_planes_any<NV>(x, a, dst);
  else
    for (int l = 0; l < a.nmod; l++) store_planes<G, NV>(x, l, dst, a.plane_stride);
}

// line-contiguous source (s_l == 1): a 32-line x 64-k tile is read along the
// lines (coalesced), turned into integers in shared memory and written along
// k: eight threads write one line's 64 contiguous residue bytes per plane.
template <bool G, class TS>
__global__ void __launch_bounds__(256, G ? 3 : 2) residues_t(const __grid_constant__ ResArgs a) {
  __shared__ double sx[2][32][65];
  const int64_t ntk = a.Kp / 64;
  const int64_t tl = blockIdx.x / ntk, tk = blockIdx.x % ntk;
  const int64_t r0 = tl * 32, kb = tk * 64;
  const int tid = threadIdx.x;
  {
    const int li = tid % 32;
    const int64_t row = r0 + li, line = a.line0 + row;
    const bool ok = row < a.lines_out && line < a.nlines && a.E[line] > -100000;
    const bool b = a.SK && *a.bal;
    double s2a = 0.0, s2b = 0.0;   // 0 -> scaled value 0 for dead lines
    if (ok && !b) line_scale(a.t, a.E[line], s2a, s2b);
    const TS *base = static_cast<const TS *>(a.base);
    double2 v[8];
#pragma unroll
    for (int jj = 0; jj < 8; jj++) {
      const int64_t k = kb + tid / 32 + jj * 8;
      v[jj] = ok && k < a.K ? ld_c(base + line + k * a.s_k) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int jj = 0; jj < 8; jj++) {
      const int j = tid / 32 + jj * 8;
      double fa = s2a, fb = s2b;
      if (ok && b) scale_pair(a.t - a.E[line] + a.sgn * a.SK[kb + j], fa, fb);
      sx[0][li][j] = scaled_magic(v[jj].x, fa, fb);
      sx[1][li][j] = scaled_magic(v[jj].y, fa, fb);
    }
  }
  __syncthreads();
  if constexpr (G) {
    // Gaussian: 16 threads per line x 4 values (64 contiguous bytes per line
    // and plane per store instruction), the 32-line tile in two halves
#pragma unroll 1
    for (int h = 0; h < 2; h++) {
      const int li = h * 16 + tid / 16, kq = (tid % 16) * 4;
      const int64_t row = r0 + li;
      if (row >= a.lines_out) break;
      ResVals<4> x;
#pragma unroll
      for (int j = 0; j < 4; j++) x.set(j, sx[0][li][kq + j], sx[1][li][kq + j]);
      gauss_planes_any<4>(x, a, a.out + row * a.Kp + kb + kq);
    }
  } else {
    const int li = tid / 8, kq = (tid % 8) * 8;
    const int64_t row = r0 + li;
    if (row >= a.lines_out) return;
    // the thread's 8 values, read from shared memory once for all moduli
    ResVals<8> x;
#pragma unroll
    for (int j = 0; j < 8; j++) x.set(j, sx[0][li][kq + j], sx[1][li][kq + j]);
    int8_t *dst = a.out + row * a.Kp + kb + kq;
    for (int l = 0; l < a.nmod; l++) store_planes<G, 8>(x, l, dst, a.plane_stride);
  }
}

// ---------------------------------------------------------------------------
// step 3: CRT reconstruction + scaling into C (complex128), O(n) and exact.
// With representatives 0 <= c_l < 3 m_l of the residues of C' and the CRT
// weights w_l = (M/m_l) ((M/m_l)^-1 mod m_l) split into three 37-bit chunks
// w_l = w_l0 + w_l1 2^37 + w_l2 2^74 (w_l2 < 2^38), the chunk sums
// S_j = sum_l c_l w_lj are exact fp64 integers (< 15 * 765 * 2^38 < 2^52) and
// X = S_0 + S_1 2^37 + S_2 2^74 == C' (mod M), 0 <= X < 15 * 765 * M. Since
// |C'| <= M/4 (choice of t), q = rint(X/M) from a double estimate is exact;
// R_j = S_j - q M_j is exact (q < 2^14, M_j < 2^38); carries normalise
// the chunks to |R_0|, |R_1| <= 2^36; C' = R_2 2^74 + R_1 2^37 + R_0 is then
// converted with ~1 ulp error.
// Guard (R26): every tile (one row, TW columns) also leaves
// sum_n |C'(m,n) 2^(-2t + E_n - max E_n)|^2 in rowsq[m * tpr + tile], the
// row's squared norm up to the factor 4^(E_m + max E_n).
// ---------------------------------------------------------------------------
struct CrtArgs {
  const uint8_t *D;         // [3n][Mc][Np], residues in [0, m)
  int64_t Mc, N, Np, m0;    // chunk rows, columns, padded columns, first row
  int nmod;
  double W[kMaxGMod][4];    // CRT weight chunks (exact integers, 37 bits each; Gaussian: 39 bits, Re weights)
  double WI[kMaxGMod][4];   // Gaussian: Im weights (39-bit chunks)
  double Cr[4], Ci[4];      // 2^XS sum_l W[l][j] (Re) and over WI (Im): offsets of the 1 + x 2^-XS encoding
  double Mch[4];            // M chunks
  double Minv;              // ~1 / M
  const int *EA, *EB;       // exponents
  int t;
  void *C;                  // double2 (complex128) or float2 (complex64, TO)
  int64_t c_sm;
  int npeer;                // peer-memory all-gather: the same element also
  void *peer[7];            // stored at peer[p] + (m c_sm + n) over NVLink
  double *rowsq;            // guard row sums [M][tpr] or null
  const int *eb_max;        // device: max_n E_n
};

template <int NCH, int CB = 37>
__device__ __forceinline__ double crt_value(const double (&S)[NCH], const double (&Mch)[4], double Minv) {
  const double two37 = (double)(1ull << CB), inv37 = 1.0 / (double)(1ull << CB);   // chunk base 2^CB
  double xe = S[NCH - 1];
#pragma unroll
  for (int j = NCH - 2; j >= 0; j--) xe = fma(xe, two37, S[j]);
  const double q = rint(xe * Minv);
  double r[NCH];
#pragma unroll
  for (int j = 0; j < NCH; j++) r[j] = fma(-q, Mch[j], S[j]);
#pragma unroll
  for (int j = 0; j < NCH - 1; j++) {
    const double cy = rint(r[j] * inv37);
    r[j] = fma(-cy, two37, r[j]);
    r[j + 1] += cy;
  }
  double x = r[NCH - 1];
#pragma unroll
  for (int j = NCH - 2; j >= 0; j--) x = fma(x, two37, r[j]);
  return x;
}

// The small representative x < 2^XS as the double 1 + x 2^-XS, built with
// integer ops only (x in the top mantissa bits of the high word): the CRT
// needs no int -> double conversion (an XU-pipe instruction that would bound
// the kernel: 30 of them per complex output against 16 XU ops / clk / SM).
// sum_l (1 + x_l 2^-XS) W_l = sum_l W_l + 2^-XS sum_l x_l W_l: every partial
// sum is a multiple of 2^-XS below 2^(53-XS), hence exact, and
// 2^XS T - 2^XS sum_l W_l recovers sum_l x_l W_l exactly.
template <int XS>
__device__ __forceinline__ double one_plus(uint32_t x) {
  return __hiloint2double((int)(0x3FF00000u | (x << (20 - XS))), 0);
}

// fixed-order block sum of one double per thread (THREADS = 32 * warps):
// xor tree inside each warp, warps in ascending order by thread 0
template <int THREADS>
__device__ __forceinline__ double block_sum_fixed(double v, double *red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < THREADS / 32; w++) s += red[w];
  return s;
}

// Persistent kernel over tiles of (one row, TW = CPT * THREADS columns). The
// 3 NMOD residue planes of a tile (3 NMOD x TW bytes) are staged in shared
// memory by cp.async.bulk (TMA) into a STAGES-deep ring completed on
// mbarriers, so later tiles' bytes are in flight while this one is reduced;
// each thread reconstructs CPT consecutive columns.
template <int CPT, int THREADS, int STAGES, int PPM = 3>
struct CrtShape {
  static constexpr int kTW = CPT * THREADS;
  static constexpr size_t smem(int nmod) { return (size_t)STAGES * PPM * nmod * kTW + 16 * STAGES; }
};

// NCH = 3 chunks while sum_l 3 m_l w_lj stays below 2^53 (nmod <= 14: top
// chunk < 2^36, sums < 2^50); 4 chunks for nmod = 15 (M > 2^117).
//
// Gaussian variant (G, R33): two planes per modulus hold c+ = phi+(C') and
// c- = phi-(C') in [0, m); Re C' = (c+ + c-) / 2 and Im C' = (c+ - c-) / (2j)
// mod m. The inverses are folded into the CRT weights (WR_l = 2^-1 w_l,
// WI_l = (2j)^-1 w_l mod M), applied to the representatives c+ + c- in
// [0, 2m) and c+ - c- + m in (0, 2m); 40-bit chunks keep every chunk sum
// exact (16 * 482 * 2^40 < 2^53) with 3 chunks for up to 16 moduli.
template <int NMOD, int NCH, int CPT, int THREADS, int STAGES, bool G, class TO>
__global__ void __launch_bounds__(THREADS + 32, 2) crt_kernel(const __grid_constant__ CrtArgs a) {
  static_assert(CPT == 2 || CPT == 4, "columns per thread");
  constexpr int PPM = G ? 2 : 3;       // planes per modulus
  constexpr int CB = G ? 39 : 37;      // CRT chunk bits
  constexpr int XS = G ? 9 : 10;       // representatives < 2^XS (Gaussian < 2m <= 482, 3M < 3m <= 765)
  using Shape = CrtShape<CPT, THREADS, STAGES, PPM>;
  constexpr int TW = Shape::kTW;
  extern __shared__ __align__(128) uint8_t crt_smem[];
  __shared__ double red[2][THREADS / 32];
  constexpr int kStage = PPM * NMOD * TW;
  // full[s]: the stage's bytes landed (TMA transaction count); empty[s]: every
  // compute warp finished reading it
  uint64_t *full = reinterpret_cast<uint64_t *>(crt_smem + STAGES * kStage);
  uint64_t *empty = full + STAGES;
  const int64_t tpr = (a.Np + TW - 1) / TW;   // tiles per row
  const int64_t ntiles = a.Mc * tpr;
  const int64_t plane = a.Mc * a.Np;
  const int tid = threadIdx.x;

  if (tid == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], THREADS / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (tid >= THREADS) {
    // producer warp: the PPM * NMOD plane rows of each tile by cp.async.bulk
    // (TMA), STAGES tiles ahead of the compute warps; it never joins their
    // barriers, so its serialized copy issue is off their critical path
    const int lane = tid - THREADS;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
      const int64_t r = tile / tpr, c0 = (tile % tpr) * TW;
      const uint32_t w = (uint32_t)(a.Np - c0 < TW ? a.Np - c0 : TW);   // multiple of 16
      if (lane == 0) {
        fence_proxy_async_smem();
        mbar_expect_tx(&full[s], PPM * NMOD * w);
      }
      __syncwarp();
      for (int q = lane; q < PPM * NMOD; q += 32)
        bulk_g2s(crt_smem + s * kStage + q * TW, a.D + q * plane + r * a.Np + c0, w, &full[s]);
    }
    return;
  }
  const int ebm = a.rowsq ? *a.eb_max : 0;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
    const int64_t r = tile / tpr, n0 = (tile % tpr) * TW + CPT * tid;
    double sq = 0.0;
    if (n0 < a.N) {
      const uint8_t *st = crt_smem + s * kStage + CPT * tid;
      double Sr[CPT][NCH], Si[CPT][NCH];
#pragma unroll
      for (int e = 0; e < CPT; e++)
#pragma unroll
        for (int j = 0; j < NCH; j++) Sr[e][j] = Si[e][j] = 0.0;
#pragma unroll
      for (int i = 0; i < NMOD; i++) {
        if constexpr (G) {
          uint32_t P, Q;
          if constexpr (CPT == 4) {
            P = *reinterpret_cast<const uint32_t *>(st + (2 * i + 0) * TW);
            Q = *reinterpret_cast<const uint32_t *>(st + (2 * i + 1) * TW);
          } else {
            P = *reinterpret_cast<const uint16_t *>(st + (2 * i + 0) * TW);
            Q = *reinterpret_cast<const uint16_t *>(st + (2 * i + 1) * TW);
          }
          const uint32_t m2 = (uint32_t)c_gmod[i] * 0x10001u;
#pragma unroll
          for (int half = 0; half < CPT / 2; half++) {
            const uint32_t sel = half ? 0x4342u : 0x4140u;
            const uint32_t p2 = __byte_perm(P, 0, sel), q2 = __byte_perm(Q, 0, sel);
            const uint32_t xr2 = p2 + q2;          // [0, 2m) per 16-bit lane
            const uint32_t xi2 = p2 + m2 - q2;     // (0, 2m)
#pragma unroll
            for (int lane = 0; lane < 2; lane++) {
              const int e = half * 2 + lane;
              const double dr = one_plus<XS>(lane ? xr2 >> 16 : xr2 & 0xffffu);
              const double di = one_plus<XS>(lane ? xi2 >> 16 : xi2 & 0xffffu);
#pragma unroll
              for (int j = 0; j < NCH; j++) {
                Sr[e][j] = fma(dr, a.W[i][j], Sr[e][j]);
                Si[e][j] = fma(di, a.WI[i][j], Si[e][j]);
              }
            }
          }
          continue;
        }
        uint32_t P, Q, S;
        if constexpr (CPT == 4) {
          P = *reinterpret_cast<const uint32_t *>(st + (3 * i + 0) * TW);
          Q = *reinterpret_cast<const uint32_t *>(st + (3 * i + 1) * TW);
          S = *reinterpret_cast<const uint32_t *>(st + (3 * i + 2) * TW);
        } else {
          P = *reinterpret_cast<const uint16_t *>(st + (3 * i + 0) * TW);
          Q = *reinterpret_cast<const uint16_t *>(st + (3 * i + 1) * TW);
          S = *reinterpret_cast<const uint16_t *>(st + (3 * i + 2) * TW);
        }
        // Unbalanced representatives, congruent to the residues of Re/Im C':
        // P - Q + m in (0, 2m), S - P - Q + 2m in (0, 3m). Computed on two 16-bit
        // lanes per register (no lane leaves [0, 2^16), so no cross-lane carry).
        const uint32_t m2 = (uint32_t)c_moduli[i] * 0x10001u;
#pragma unroll
        for (int half = 0; half < CPT / 2; half++) {
          const uint32_t sel = half ? 0x4342u : 0x4140u;
          const uint32_t p2 = __byte_perm(P, 0, sel), q2 = __byte_perm(Q, 0, sel), s2 = __byte_perm(S, 0, sel);
          const uint32_t cr2 = p2 + m2 - q2;
          const uint32_t ci2 = s2 + 2u * m2 - p2 - q2;
#pragma unroll
          for (int lane = 0; lane < 2; lane++) {
            const int e = half * 2 + lane;
            const double dr = one_plus<XS>(lane ? cr2 >> 16 : cr2 & 0xffffu);
            const double di = one_plus<XS>(lane ? ci2 >> 16 : ci2 & 0xffffu);
#pragma unroll
            for (int j = 0; j < NCH; j++) {
              Sr[e][j] = fma(dr, a.W[i][j], Sr[e][j]);
              Si[e][j] = fma(di, a.WI[i][j], Si[e][j]);
            }
          }
        }
      }
      // undo the 1 + x 2^-XS encoding: S_j = 2^XS T_j - 2^XS sum_l W_lj (exact)
#pragma unroll
      for (int e = 0; e < CPT; e++)
#pragma unroll
        for (int j = 0; j < NCH; j++) {
          Sr[e][j] = fma(Sr[e][j], (double)(1 << XS), -a.Cr[j]);
          Si[e][j] = fma(Si[e][j], (double)(1 << XS), -a.Ci[j]);
        }
      const int64_t m = a.m0 + r;
      const int ea = a.EA[m];
      const int sc0 = -(2 * a.t - ea);
#pragma unroll
      for (int e = 0; e < CPT; e++) {
        const int64_t n = n0 + e;
        if (n >= a.N) break;
        const int eb = a.EB[n];
        double2 out = make_double2(0.0, 0.0);
        if (ea > -100000 && eb > -100000) {
          const double xr = crt_value<NCH, CB>(Sr[e], a.Mch, a.Minv);
          const double xi = crt_value<NCH, CB>(Si[e], a.Mch, a.Minv);
          const int sc = sc0 + eb;
          if (sc >= -1022 && sc <= 1023) {   // 2^sc is a normal double: one exact multiply
            const double f = __hiloint2double((sc + 1023) << 20, 0);
            out = make_double2(xr * f, xi * f);
          } else {
            out = make_double2(ldexp(xr, sc), ldexp(xi, sc));
          }
          if (a.rowsq) {
            const double g = pow2i(-2 * a.t + eb - ebm);
            sq = fma(xr * g, xr * g, sq);
            sq = fma(xi * g, xi * g, sq);
          }
        }
        st_c(static_cast<TO *>(a.C) + m * a.c_sm + n, out);
#pragma unroll 1
        for (int pp = 0; pp < a.npeer; pp++) st_c(static_cast<TO *>(a.peer[pp]) + m * a.c_sm + n, out);
      }
    }
    if (a.rowsq) {
      // deterministic tile sum; red is double-buffered across iterations
      double v = sq;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((tid & 31) == 0) red[it & 1][tid >> 5] = v;
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);   // this warp is done with stage s
    if (a.rowsq) {
      named_bar_sync(1, THREADS);                   // compute warps only
      if (tid == 0) {
        double v = 0.0;
        for (int w = 0; w < THREADS / 32; w++) v += red[it & 1][w];
        a.rowsq[(a.m0 + tile / tpr) * tpr + tile % tpr] = v;
      }
    }
  }
}

template <int NMOD, int NCH, int CPT, int THREADS, int STAGES, bool G, class TO>
cudaError_t launch_crt_cfg(const CrtArgs &c, int64_t mc, cudaStream_t s) {
  using Shape = CrtShape<CPT, THREADS, STAGES, G ? 2 : 3>;
  auto kern = crt_kernel<NMOD, NCH, CPT, THREADS, STAGES, G, TO>;
  const size_t smem = Shape::smem(NMOD);
  cudaError_t e = ensure_smem_attr((const void *)kern, smem);
  if (e != cudaSuccess) return e;
  const int sms = device_sms(), per_sm = occupancy_per_sm((const void *)kern, THREADS + 32, smem);
  const int64_t ntiles = mc * ((c.Np + Shape::kTW - 1) / Shape::kTW);
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)std::max(per_sm, 1) * sms);
  kern<<<grid, THREADS + 32, smem, s>>>(c);   // + the producer warp
  return cudaGetLastError();
}

constexpr int kCrtTW = 1024;   // CRT tile width (columns): 4 per thread x 256 threads
// 4 columns x 256 threads x 2 stages: measured best of {2,4} x {128,256} x
// {2,3,4} on the target shapes (the kernel is XU/FP64-issue bound there).
template <int NMOD, int NCH, bool G, class TO>
cudaError_t launch_crt(const CrtArgs &c, int64_t mc, cudaStream_t s) {
  // Gaussian stages are 2/3 the size of 3M ones: three fit beside a second CTA
  // (2 columns x 512 threads measured slower: 6.82 vs 6.46 ms per apply)
  return launch_crt_cfg<NMOD, NCH, 4, 256, G ? 3 : 2, G, TO>(c, mc, s);
}

// ---------------------------------------------------------------------------
// float64 (real) Ozaki-II: one residue plane per modulus (no 3M split), the
// same scaling, moduli, INT8 GEMM + mod-m epilogue and CRT; n GEMMs instead
// of 3n. C'(m, n) = sum_k A'(m, k) B'(k, n) with |C'| <= K 2^(2t) <= M/8.
// ---------------------------------------------------------------------------
// K-contiguous: 8 consecutive k of one line per thread, 8 bytes per plane
template <class TS>
__global__ void __launch_bounds__(256) residues_real(const __grid_constant__ ResArgs a) {
  const int64_t kgroups = a.Kp / 8;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= a.lines_out * kgroups) return;
  const int64_t row = gid / kgroups, k0 = (gid % kgroups) * 8, line = a.line0 + row;
  double x[8];
  int lo[8];
  if (line < a.nlines && a.E[line] > -100000) {
    const TS *p = static_cast<const TS *>(a.base) + line * a.s_l;
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) v[j] = k0 + j < a.K ? ld_r(p + (k0 + j) * a.s_k) : 0.0;
    double fa[8], fb[8];
    if (a.SK && *a.bal) {
      elem_scales(a, a.E[line], k0, fa, fb);
    } else {
      double s2a, s2b;
      line_scale(a.t, a.E[line], s2a, s2b);
#pragma unroll
      for (int j = 0; j < 8; j++) {
        fa[j] = s2a;
        fb[j] = s2b;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const double m = scaled_magic(v[j], fa[j], fb[j]);
      x[j] = m - kMagic;
      lo[j] = __double2loint(m);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      x[j] = 0.0;
      lo[j] = 0;
    }
  }
  int8_t *dst = a.out + row * a.Kp + k0;
  for (int l = 0; l < a.nmod; l++) {
    const int mi = c_moduli[l];
    const double minv = c_minv[l];
    int r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = bal_res(x[j], lo[j], minv, mi);
    *reinterpret_cast<uint2 *>(dst + (int64_t)l * a.plane_stride) =
        make_uint2(pack4(r[0], r[1], r[2], r[3]), pack4(r[4], r[5], r[6], r[7]));
  }
}

// line-contiguous: 32-line x 64-k tile through shared memory (as residues_t)
template <class TS>
__global__ void __launch_bounds__(256) residues_real_t(const __grid_constant__ ResArgs a) {
  __shared__ double sx[32][65];
  const int64_t ntk = a.Kp / 64;
  const int64_t tl = blockIdx.x / ntk, tk = blockIdx.x % ntk;
  const int64_t r0 = tl * 32, kb = tk * 64;
  const int tid = threadIdx.x;
  {
    const int li = tid % 32;
    const int64_t row = r0 + li, line = a.line0 + row;
    const bool ok = row < a.lines_out && line < a.nlines && a.E[line] > -100000;
    const bool b = a.SK && *a.bal;
    double s2a = 0.0, s2b = 0.0;
    if (ok && !b) line_scale(a.t, a.E[line], s2a, s2b);
    const TS *base = static_cast<const TS *>(a.base);
    double v[8];
#pragma unroll
    for (int jj = 0; jj < 8; jj++) {
      const int64_t k = kb + tid / 32 + jj * 8;
      v[jj] = ok && k < a.K ? ld_r(base + line + k * a.s_k) : 0.0;
    }
#pragma unroll
    for (int jj = 0; jj < 8; jj++) {
      const int j = tid / 32 + jj * 8;
      double fa = s2a, fb = s2b;
      if (ok && b) scale_pair(a.t - a.E[line] + a.sgn * a.SK[kb + j], fa, fb);
      sx[li][j] = scaled_magic(v[jj], fa, fb);
    }
  }
  __syncthreads();
  const int li = tid / 8, kq = (tid % 8) * 8;
  const int64_t row = r0 + li;
  if (row >= a.lines_out) return;
  double x[8];
  int lo[8];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const double m = sx[li][kq + j];
    x[j] = m - kMagic;
    lo[j] = __double2loint(m);
  }
  int8_t *dst = a.out + row * a.Kp + kb + kq;
  for (int l = 0; l < a.nmod; l++) {
    const int mi = c_moduli[l];
    const double minv = c_minv[l];
    int r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = bal_res(x[j], lo[j], minv, mi);
    *reinterpret_cast<uint2 *>(dst + (int64_t)l * a.plane_stride) =
        make_uint2(pack4(r[0], r[1], r[2], r[3]), pack4(r[4], r[5], r[6], r[7]));
  }
}

// CRT for real outputs: the residue of C' modulo m_l is the GEMM's byte in
// [0, m_l) itself; 4 consecutive columns per thread (one 32-bit load per
// plane); block b covers row b / tpr, columns (b % tpr) * 1024 + [0, 1024)
struct CrtArgsR {
  const uint8_t *D;          // [n][Mc][Np]
  int64_t Mc, N, Np, m0;
  int nmod;
  double W[kMaxMod][4];
  double C0[4];              // 2^8 sum_l W[l][j] (one_plus<8> encoding offset)
  double Mch[4];
  double Minv;
  const int *EA, *EB;
  int t;
  void *C;                   // double or float (TO)
  int64_t c_sm;
  double *rowsq;             // guard row sums [M][tpr] or null
  const int *eb_max;
};

template <int NMOD, int NCH, class TO>
__global__ void __launch_bounds__(256) crt_real_kernel(const __grid_constant__ CrtArgsR a) {
  __shared__ double red[8];
  const int64_t tpr = (a.Np + kCrtTW - 1) / kCrtTW;
  const int64_t r = blockIdx.x / tpr, tile = blockIdx.x % tpr;
  const int64_t n0 = tile * kCrtTW + 4 * threadIdx.x;
  const int64_t plane = a.Mc * a.Np;
  const int64_t m = a.m0 + r;
  double sq = 0.0;
  if (n0 < a.N) {
    double S[4][NCH];
#pragma unroll
    for (int e = 0; e < 4; e++)
#pragma unroll
      for (int j = 0; j < NCH; j++) S[e][j] = 0.0;
#pragma unroll
    for (int i = 0; i < NMOD; i++) {
      const uint32_t w4 = __ldg(reinterpret_cast<const uint32_t *>(a.D + i * plane + r * a.Np + n0));
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const double c = one_plus<8>((w4 >> (8 * e)) & 0xffu);   // 1 + byte 2^-8, no I2F
#pragma unroll
        for (int j = 0; j < NCH; j++) S[e][j] = fma(c, a.W[i][j], S[e][j]);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; e++)
#pragma unroll
      for (int j = 0; j < NCH; j++) S[e][j] = fma(S[e][j], 256.0, -a.C0[j]);
    const int ea = a.EA[m];
    const int ebm = a.rowsq ? *a.eb_max : 0;
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int64_t n = n0 + e;
      if (n >= a.N) break;
      const int eb = a.EB[n];
      double out = 0.0;
      if (ea > -100000 && eb > -100000) {
        const double x = crt_value(S[e], a.Mch, a.Minv);
        const int sc = -(2 * a.t - ea) + eb;
        out = (sc >= -1022 && sc <= 1023) ? x * __hiloint2double((sc + 1023) << 20, 0) : ldexp(x, sc);
        if (a.rowsq) {
          const double g = pow2i(-2 * a.t + eb - ebm);
          sq = fma(x * g, x * g, sq);
        }
      }
      st_r(static_cast<TO *>(a.C) + m * a.c_sm + n, out);
    }
  }
  if (a.rowsq) {
    const double v = block_sum_fixed<256>(sq, red);
    if (threadIdx.x == 0) a.rowsq[m * tpr + tile] = v;
  }
}

// ---------------------------------------------------------------------------
// Accuracy guard (R26). Operand entry (m, k) of A is rounded to an
// integer at scale 2^(t - E_m + s_k): its error is eps 2^(E_m - t - s_k) with
// eps uniform in [-1/2, 1/2] per real component, so (independent errors)
//   E ||C~ - AB||_F^2 = c 4^-t (S_M ||B'||_F^2 + ||A'||_F^2 S_N),
// S_M = sum_m 4^E_m, S_N = sum_n 4^E_n, A' = A diag(2^s), B' = diag(2^-s) B,
// c = 1/6 (complex: two components) or 1/12 (real). The kernel compares
// est = sqrt(that) with tol ||C~||_F and sets the recomputation flag. All
// sums are normalised by 4^max E (no overflow) and taken in a fixed order.
// Without per-k statistics of A (A streamed in row chunks) ||A'||^2 is
// bounded by (2) K S_M.
// ---------------------------------------------------------------------------
struct GuardArgs {
  const int *EA, *EB;
  int64_t M, N, K, tpr;
  const int *KA, *KB, *SK;     // KA may be null
  const double *KSA, *KSB;     // KSA null with KA
  const double *rowsq;
  int t, cplx;
  double tol;
  int *flag;                   // out: 1 = recompute on DMMA
  int *bal;                    // balancing was active
  OzGuard *rec;                // optional statistics
};

// rowsq[m][0] = sum_j rowsq[m][j]: warp per row, the slots read coalesced
// and summed in a fixed order (lane-strided partials, then an xor tree)
__global__ void __launch_bounds__(256) rowsq_fold(double *rowsq, int64_t M, int64_t tpr) {
  const int lane = threadIdx.x & 31;
  for (int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; m < M;
       m += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double r = 0.0;
    for (int64_t j = lane; j < tpr; j += 32) r += rowsq[m * tpr + j];
#pragma unroll
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    __syncwarp();
    if (lane == 0) rowsq[m * tpr] = r;
  }
}

__global__ void __launch_bounds__(1024) guard_finalize(const __grid_constant__ GuardArgs g) {
  __shared__ double red[32];
  const int tid = threadIdx.x;
  auto bsum = [&](double v) -> double {   // fixed-order block sum, result broadcast
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
    return s;
  };
  auto bmax = [&](const int *E, int64_t n) -> int {
    int v = -100000;
    for (int64_t i = tid; i < n; i += blockDim.x) v = max(v, E[i]);
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = (double)v;
    __syncthreads();
    double s = -100000.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s = fmax(s, red[w]);
    return (int)s;
  };
  const int ea = bmax(g.EA, g.M);
  const int eb = bmax(g.EB, g.N);
  double sM = 0.0, sN = 0.0, nA = 0.0, nB = 0.0, nC = 0.0;
  // row sums: slot 0 of each row (rowsq_fold ran first when tpr > 1)
  for (int64_t m = tid; m < g.M; m += blockDim.x) {
    const int e = g.EA[m];
    if (e == -100000) continue;
    const double w = pow4i(e - ea);
    sM += w;
    nC = fma(w, g.rowsq[m * g.tpr], nC);
  }
  for (int64_t n = tid; n < g.N; n += blockDim.x)
    if (g.EB[n] != -100000) sN += pow4i(g.EB[n] - eb);
  for (int64_t k = tid; k < g.K; k += blockDim.x) {
    const int s = g.SK ? g.SK[k] : 0;
    if (g.KA && g.KA[k] != -100000) nA = fma(g.KSA[k], pow4i(g.KA[k] + s - ea), nA);
    if (g.KB[k] != -100000) nB = fma(g.KSB[k], pow4i(g.KB[k] - s - eb), nB);
  }
  sM = bsum(sM);
  sN = bsum(sN);
  nC = bsum(nC);
  nB = bsum(nB);
  nA = g.KA ? bsum(nA) : (g.cplx ? 2.0 : 1.0) * (double)g.K * sM;
  if (tid == 0) {
    int fall = 0;
    double est = 0.0;
    if (ea != -100000 && eb != -100000) {
      // 4^-t applied as (2^-t)^2 on the normalised sums
      const double c = g.cplx ? 1.0 / 6.0 : 1.0 / 12.0;
      const double e2 = c * (sM * nB + nA * sN);
      const double st = ldexp(1.0, -g.t);
      const double errn = sqrt(e2) * st;   // ||dC|| / 2^(ea + eb)
      const double cn = sqrt(nC);          // ||C|| / 2^(ea + eb)
      est = cn > 0.0 ? errn / cn : (errn > 0.0 ? INFINITY : 0.0);
      fall = !(est <= g.tol);
    }
    *g.flag = fall;
    if (g.rec) {
      g.rec->gemms++;
      g.rec->fallbacks += fall;
      g.rec->balanced += (g.bal && *g.bal) ? 1 : 0;
      g.rec->last_est = est;
      if (!(est <= g.rec->max_est)) g.rec->max_est = est;
    }
  }
}

// the guard's recomputation also reaches the peers' copies of the slab
// (fused all-gather): C rows [0, M) with row stride c_sm, copied to the same
// offsets of every peer buffer when *run_if != 0
struct PeerSet {
  double2 *p[7];
};
__global__ void __launch_bounds__(256) copy_to_peers_if(const double2 *C, int64_t M, int64_t N, int64_t c_sm, int np,
                                                       const __grid_constant__ PeerSet ps, const int *run_if) {
  if (*reinterpret_cast<const volatile int *>(run_if) == 0) return;
  double2 *const *pp = ps.p;
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / N, n = i % N;
    const double2 v = C[m * c_sm + n];
    for (int p = 0; p < np; p++) pp[p][m * c_sm + n] = v;
  }
}

// ---------------------------------------------------------------------------
// host planning
// ---------------------------------------------------------------------------
// scratch budget of the residue planes + byte outputs of one row chunk
// (8 GB; TCI_OZ_CHUNK_GB overrides, read once)
size_t oz_budget() {
  static const size_t b = [] {
    const char *e = std::getenv("TCI_OZ_CHUNK_GB");
    const long v = e ? std::atol(e) : 0;
    return (size_t)(v > 0 && v <= 64 ? v : 8) << 30;
  }();
  return b;
}

// moduli sets: 3M complex and real (kModuli), Gaussian complex (kGModuli)
enum OzKind { kOzReal = 0, kOz3M = 1, kOzGauss = 2 };

struct OzPlan {
  int kind, nmod, t, ppm;   // ppm: residue planes per modulus (1 real, 3 3M, 2 Gaussian)
  int64_t Kp, Np, Mc, chunks, tpr, nch;
  size_t off_EA, off_EB, off_Bres, off_Ares, off_D;
  size_t off_KA, off_KB, off_SK, off_KSA, off_KSB, off_slotE, off_slotS, off_rowsq, off_misc;
  size_t total;
};

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
size_t align_up(size_t x) { return (x + 255) / 256 * 256; }

// exactness (R26/R33): |C'| <= 2 K 2^(2t) <= M/4, i.e. 2t + 3 + log2 K <= log2 M;
// the fewest moduli that allow t >= tmin (46 for float64 sources, 24 for
// float32: R34), then the largest such t
bool crt_mma_enabled();
OzPlan oz_plan(int64_t M, int64_t N, int64_t K, size_t budget_D, int64_t max_rows = 0, int kind = kOz3M,
               int tmin = 46) {
  OzPlan p{};
  p.kind = kind;
  p.ppm = kind == kOzReal ? 1 : kind == kOz3M ? 3 : 2;
  const int *mods = kind == kOzGauss ? kGModuli : kModuli;
  const int nmax = kind == kOzGauss ? kMaxGMod : kMaxMod;
  const double lk = std::log2((double)std::max<int64_t>(K, 1));
  double lm = 0;
  p.nmod = 0;
  for (int l = 0; l < nmax; l++) {
    lm += std::log2((double)mods[l]);
    p.nmod = l + 1;
    if (std::floor((lm - 3.0 - lk) / 2.0) >= tmin) break;
  }
  p.t = (int)std::floor((lm - 3.0 - lk) / 2.0);
  p.Kp = round_up(K, 64);
  p.Np = round_up(N, 16);
  const int64_t planes = p.ppm * p.nmod;
  // rows per chunk: uint8 residue outputs + A residues within budget_D, multiple of 256
  int64_t mc = (int64_t)(budget_D / ((size_t)planes * (p.Np + p.Kp)));
  mc = std::max<int64_t>(256, mc / 256 * 256);
  p.Mc = std::min<int64_t>(round_up(M, 256), mc);
  if (max_rows > 0) p.Mc = std::min<int64_t>(p.Mc, std::max<int64_t>(256, round_up(max_rows, 256)));
  p.chunks = (M + p.Mc - 1) / p.Mc;
  p.tpr = (kind == kOzGauss || kind == kOzReal) && crt_mma_enabled() ? crt_mma_slots_per_row(p.Np)
                                                                    : (p.Np + kCrtTW - 1) / kCrtTW;
  p.nch = std::max<int64_t>(1, std::min<int64_t>(64, ((int64_t)1 << 22) / p.Kp));
  size_t off = 0;
  p.off_EA = off; off = align_up(off + (size_t)M * 4);
  p.off_EB = off; off = align_up(off + (size_t)N * 4);
  p.off_Bres = off; off = align_up(off + (size_t)planes * p.Np * p.Kp);
  p.off_Ares = off; off = align_up(off + (size_t)planes * p.Mc * p.Kp);
  p.off_D = off; off = align_up(off + (size_t)planes * p.Mc * p.Np);
  p.off_KA = off; off = align_up(off + (size_t)p.Kp * 4);
  p.off_KB = off; off = align_up(off + (size_t)p.Kp * 4);
  p.off_SK = off; off = align_up(off + (size_t)p.Kp * 4);
  p.off_KSA = off; off = align_up(off + (size_t)p.Kp * 8);
  p.off_KSB = off; off = align_up(off + (size_t)p.Kp * 8);
  p.off_slotE = off; off = align_up(off + (size_t)p.nch * p.Kp * 4);
  p.off_slotS = off; off = align_up(off + (size_t)p.nch * p.Kp * 8);
  p.off_rowsq = off; off = align_up(off + (size_t)M * p.tpr * 8);
  p.off_misc = off; off = align_up(off + 64);
  p.total = off;
  return p;
}

// modular helpers on the host (unsigned 128-bit)
typedef unsigned __int128 u128;
u128 mulmod_small(u128 a, unsigned b, u128 M) {   // (a * b) mod M, a < M < 2^126, b < 256
  u128 r = 0;
  for (int bit = 7; bit >= 0; bit--) {
    r = (r << 1) % M;
    if (b >> bit & 1) r = (r + a) % M;
  }
  return r;
}
// modular inverse on the host (extended Euclid)
unsigned inv_mod(unsigned a, unsigned m) {
  int t = 0, nt = 1, r = (int)m, nr = (int)(a % m);
  while (nr) {
    const int q = r / nr;
    int tmp = t - q * nt; t = nt; nt = tmp;
    tmp = r - q * nr; r = nr; nr = tmp;
  }
  return (unsigned)(t < 0 ? t + (int)m : t);
}

// CRT weight chunks (37 bits each), M chunks and ~1/M for nmod moduli
void crt_constants(int nmod, double (&W)[kMaxMod][4], double (&Mch)[4], double &Minv) {
  u128 Mp = 1;
  for (int l = 0; l < nmod; l++) Mp *= (u128)kModuli[l];
  const u128 mask = ((u128)1 << 37) - 1;
  for (int l = 0; l < nmod; l++) {
    const unsigned ml = (unsigned)kModuli[l];
    const u128 Ml = Mp / ml;
    const u128 wl = mulmod_small(Ml, inv_mod((unsigned)(Ml % ml), ml), Mp);
    for (int j = 0; j < 4; j++) W[l][j] = (double)(uint64_t)((wl >> (37 * j)) & mask);
  }
  for (int j = 0; j < 4; j++) Mch[j] = (double)(uint64_t)((Mp >> (37 * j)) & mask);
  Minv = 1.0 / ((double)(uint64_t)(Mp >> 64) * 18446744073709551616.0 + (double)(uint64_t)Mp);
}

// Gaussian set (R33): WR_l = (2^-1 mod m_l) w_l mod M and WI_l = ((2 j_l)^-1
// mod m_l) w_l mod M in 39-bit chunks (3 chunks for 15 moduli, M < 2^112;
// 4 for 16), M chunks, ~1/M
constexpr int kGaussCB = 39;
void crt_constants_gauss(int nmod, double (&WR)[kMaxGMod][4], double (&WI)[kMaxGMod][4], double (&Mch)[4],
                         double &Minv) {
  u128 Mp = 1;
  for (int l = 0; l < nmod; l++) Mp *= (u128)kGModuli[l];
  const u128 mask = ((u128)1 << kGaussCB) - 1;
  for (int l = 0; l < kMaxGMod; l++)
    for (int j = 0; j < 4; j++) WR[l][j] = WI[l][j] = 0.0;
  for (int l = 0; l < nmod; l++) {
    const unsigned ml = (unsigned)kGModuli[l];
    const u128 Ml = Mp / ml;
    const u128 wl = mulmod_small(Ml, inv_mod((unsigned)(Ml % ml), ml), Mp);
    const unsigned h = inv_mod(2u, ml);
    const unsigned jl = (unsigned)((kGRoots[l] % (int)ml + (int)ml) % (int)ml);
    const unsigned g = inv_mod((2u * jl) % ml, ml);
    const u128 wr = mulmod_small(wl, h, Mp), wi = mulmod_small(wl, g, Mp);
    for (int j = 0; j < 4; j++) {
      WR[l][j] = (double)(uint64_t)((wr >> (kGaussCB * j)) & mask);
      WI[l][j] = (double)(uint64_t)((wi >> (kGaussCB * j)) & mask);
    }
  }
  for (int j = 0; j < 4; j++) Mch[j] = (double)(uint64_t)((Mp >> (kGaussCB * j)) & mask);
  Minv = 1.0 / ((double)(uint64_t)(Mp >> 64) * 18446744073709551616.0 + (double)(uint64_t)Mp);
}

// The tensor-core CRT (crt_mma.cu, default; TCI_CRT_MMA=0 keeps crt_kernel):
// digit matrix Bd[k][j] (plane k = 2l: c+_l, 2l + 1: c-_l; columns 0..15 the
// base-256 digits of WR_l, 16..31 those of WI_l for c+ and of M - WI_l for
// c-), 32-bit chunks of M, ~1/M
bool crt_mma_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("TCI_CRT_MMA");
    return !(e && e[0] == '0');
  }();
  return on;
}
void crt_digits_gauss(int nmod, CrtMmaArgs &c) {
  u128 Mp = 1;
  for (int l = 0; l < nmod; l++) Mp *= (u128)kGModuli[l];
  for (int k = 0; k < 32; k++)
    for (int j = 0; j < 32; j++) c.Bd[k][j] = 0;
  for (int l = 0; l < nmod; l++) {
    const unsigned ml = (unsigned)kGModuli[l];
    const u128 Ml = Mp / ml;
    const u128 wl = mulmod_small(Ml, inv_mod((unsigned)(Ml % ml), ml), Mp);
    const unsigned h = inv_mod(2u, ml);
    const unsigned jl = (unsigned)((kGRoots[l] % (int)ml + (int)ml) % (int)ml);
    const unsigned g = inv_mod((2u * jl) % ml, ml);
    const u128 wr = mulmod_small(wl, h, Mp), wi = mulmod_small(wl, g, Mp);
    const u128 wim = wi ? Mp - wi : 0;
    for (int j = 0; j < 16; j++) {
      c.Bd[2 * l][j] = c.Bd[2 * l + 1][j] = (uint8_t)(wr >> (8 * j));
      c.Bd[2 * l][16 + j] = (uint8_t)(wi >> (8 * j));
      c.Bd[2 * l + 1][16 + j] = (uint8_t)(wim >> (8 * j));
    }
  }
  int bits = 0;
  for (u128 x = Mp; x; x >>= 1) bits++;
  c.nd = (bits + 7) / 8;
  c.planes = 2 * nmod;
  for (int j = 0; j < 4; j++) c.Mch[j] = (double)(uint64_t)((Mp >> (32 * j)) & 0xFFFFFFFFu);
  // 2^(32 (NC - 2)) / M, NC = the 32-bit chunks the epilogue uses (crt_mma.cu)
  const int nc = ((c.nd + 1) / 2 + 1) / 2;
  c.Minv = std::ldexp(1.0, 32 * (nc - 2)) / ((double)(uint64_t)(Mp >> 64) * 18446744073709551616.0 + (double)(uint64_t)Mp);
}

// real outputs: plane l holds c_l = C' mod m_l (moduli kModuli); columns
// 0..15 the base-256 digits of the CRT weight w_l, 16..31 zero
void crt_digits_real(int nmod, CrtMmaArgs &c) {
  u128 Mp = 1;
  for (int l = 0; l < nmod; l++) Mp *= (u128)kModuli[l];
  for (int k = 0; k < 32; k++)
    for (int j = 0; j < 32; j++) c.Bd[k][j] = 0;
  for (int l = 0; l < nmod; l++) {
    const unsigned ml = (unsigned)kModuli[l];
    const u128 Ml = Mp / ml;
    const u128 wl = mulmod_small(Ml, inv_mod((unsigned)(Ml % ml), ml), Mp);
    for (int j = 0; j < 16; j++) c.Bd[l][j] = (uint8_t)(wl >> (8 * j));
  }
  int bits = 0;
  for (u128 x = Mp; x; x >>= 1) bits++;
  c.nd = (bits + 7) / 8;
  c.planes = nmod;
  for (int j = 0; j < 4; j++) c.Mch[j] = (double)(uint64_t)((Mp >> (32 * j)) & 0xFFFFFFFFu);
  const int nc = ((c.nd + 1) / 2 + 1) / 2;
  c.Minv = std::ldexp(1.0, 32 * (nc - 2)) / ((double)(uint64_t)(Mp >> 64) * 18446744073709551616.0 + (double)(uint64_t)Mp);
}

// one batched INT8 GEMM: D[b][m][n] = (sum_k A[b][m][k] B[b][n][k]) mod m_b
// (i8gemm.cu: hand-written tcgen05 kind::i8, TMA, TMEM)
cudaError_t int8_gemm(const GemmProblem &g, const OzPlan &p, const int8_t *Ares, const int8_t *Bres, uint8_t *D,
                      int64_t mc, int planes, int per_mod, int *counter, cudaStream_t s, int64_t *launches) {
  OzProf *pf = g.oz_prof;
  const bool rec = pf && pf->n < 64;
  if (rec) {
    cudaEventCreate(&pf->a[pf->n]);
    cudaEventCreate(&pf->b[pf->n]);
    cudaEventRecord(pf->a[pf->n], s);
  }
  cudaError_t e = launch_i8gemm(Ares, Bres, D, mc, p.Np, p.Kp, planes, per_mod,
                                p.kind == kOzGauss ? kGModuli : kModuli, p.nmod, counter, s, launches);
  if (e != cudaSuccess) return e;
  if (rec) {
    cudaEventRecord(pf->b[pf->n], s);
    pf->ops[pf->n] = 2.0 * (double)mc * p.Np * p.Kp * planes;
    pf->n++;
  }
  return cudaSuccess;
}

// Shared prologue / epilogue of the complex and real Ozaki GEMMs: per-k
// statistics and K-balancing (step 0), exponents (step 1a), and after the
// chunks the guard and its DMMA recomputation.
template <class T>
struct OzRun {
  const GemmProblem &g;
  const OzPlan &p;
  char *w;
  cudaStream_t s;
  int64_t *launches;
  int *EA, *EB, *KA, *KB, *SK, *misc;
  double *KSA, *KSB, *rowsq;
  bool guard, staged, have_ka;
  int64_t a_sm, a_sk, b_sk, b_sn;

  OzRun(const GemmProblem &g_, const OzPlan &p_, void *ws, cudaStream_t s_, int64_t *l_)
      : g(g_), p(p_), w(static_cast<char *>(ws)), s(s_), launches(l_) {
    EA = reinterpret_cast<int *>(w + p.off_EA);
    EB = reinterpret_cast<int *>(w + p.off_EB);
    KA = reinterpret_cast<int *>(w + p.off_KA);
    KB = reinterpret_cast<int *>(w + p.off_KB);
    SK = reinterpret_cast<int *>(w + p.off_SK);
    KSA = reinterpret_cast<double *>(w + p.off_KSA);
    KSB = reinterpret_cast<double *>(w + p.off_KSB);
    rowsq = reinterpret_cast<double *>(w + p.off_rowsq);
    misc = reinterpret_cast<int *>(w + p.off_misc);   // [0] fallback flag, [1] balancing, [2] max E_n, [3] tile counter
    guard = g.oz_tol > 0.0;
    staged = g.rows_needed != nullptr;
    a_sk = g.K == 1 ? 1 : g.a_sk;
    a_sm = g.a_sm;
    b_sk = g.b_sk;
    b_sn = g.N == 1 ? 1 : g.b_sn;
    have_ka = false;
  }
  void count(int n = 1) {
    if (launches) *launches += n;
  }
  // per-k statistics over the lines of X: element (l, k) at l*s_l + k*s_k
  // fused variant: also the unbalanced line exponents E (pre-filled with
  // -100000 here); returns false when it does not apply (E untouched)
  bool kstats_lx(const T *X, int64_t L, int64_t s_l, int64_t s_k, int *KE, double *KS, int *E) {
    int *SE = reinterpret_cast<int *>(w + p.off_slotE);
    double *SS = reinterpret_cast<double *>(w + p.off_slotS);
    // line chunks: >= 64 lines per (k-block, chunk) for the thread-per-k
    // variant (as kstats_cols), up to 4096 for the warp-per-k one; their line
    // maxima live in shared memory
    const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(p.nch, s_l == 1 ? (L + 4095) / 4096 : (L + 63) / 64));
    const int64_t chunk = (L + nch - 1) / nch;
    if (s_l != 1 && s_k != 1) return false;
    if (chunk * 4 > 48 * 1024) return false;   // shared line maxima of one chunk
    fill_int<<<(unsigned)std::min<int64_t>((L + 255) / 256, 1024), 256, 0, s>>>(E, L, -100000);
    if (s_l == 1) {
      dim3 grid((unsigned)((g.K + 31) / 32), (unsigned)nch);
      kstats_lines_lx<T><<<grid, 256, (size_t)chunk * 4, s>>>(X, g.K, L, s_k, chunk, SE, SS, E);
    } else {
      dim3 grid((unsigned)((g.K + 255) / 256), (unsigned)nch);
      kstats_cols_lx<T><<<grid, 256, (size_t)chunk * 4, s>>>(X, g.K, L, s_l, chunk, SE, SS, E);
    }
    kstats_merge<<<(unsigned)((g.K + 255) / 256), 256, 0, s>>>(SE, SS, (int)nch, g.K, KE, KS);
    count(3);
    return true;
  }
  void kstats(const T *X, int64_t L, int64_t s_l, int64_t s_k, int *KE, double *KS) {
    if (s_l == 1) {
      kstats_lines<T><<<(unsigned)((g.K * 32 + 255) / 256), 256, 0, s>>>(X, g.K, L, s_k, KE, KS);
      count();
    } else {
      int *SE = reinterpret_cast<int *>(w + p.off_slotE);
      double *SS = reinterpret_cast<double *>(w + p.off_slotS);
      const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(p.nch, (L + 63) / 64));
      const int64_t chunk = (L + nch - 1) / nch;
      dim3 grid((unsigned)((g.K + 255) / 256), (unsigned)nch);
      kstats_cols<T><<<grid, 256, 0, s>>>(X, g.K, L, s_l, chunk, SE, SS);
      kstats_merge<<<(unsigned)((g.K + 255) / 256), 256, 0, s>>>(SE, SS, (int)nch, g.K, KE, KS);
      count(2);
    }
  }
  // only_if_bal: E already holds the unbalanced exponents (fused stats
  // pass); recompute only when the device flag says the balancing is on
  void exponents(const T *X, int64_t nl, int64_t s_l, int64_t s_k, int *E, int sgn, bool only_if_bal = false) {
    const int oib = only_if_bal ? 1 : 0;
    if (s_k == 1) {
      line_exponent<T><<<(unsigned)((nl * 32 + 255) / 256), 256, 0, s>>>(X, nl, g.K, s_l, s_k, E, SK, sgn, misc + 1,
                                                                         oib);
      count();
    } else {
      fill_int<<<(unsigned)std::min<int64_t>((nl + 255) / 256, 1024), 256, 0, s>>>(E, nl, -100000,
                                                                                   only_if_bal ? misc + 1 : nullptr);
      const int64_t ky = std::max<int64_t>(1, std::min<int64_t>((g.K + 127) / 128, 65535));
      dim3 grid((unsigned)((nl + 255) / 256), (unsigned)ky);
      line_exponent<T><<<grid, 256, 0, s>>>(X, nl, g.K, s_l, s_k, E, SK, sgn, misc + 1, oib);
      count(2);
    }
  }
  // steps 0 and 1a for B (and A unless it streams in by row chunks)
  void prologue() {
    const T *A = static_cast<const T *>(g.A), *B = static_cast<const T *>(g.B);
    const bool bal = g.oz_balance && !staged;
    bool fusedB = false, fusedA = false;   // E from the statistics pass
    if (bal || guard) fusedB = kstats_lx(B, g.N, b_sn, b_sk, KB, KSB, EB) || (kstats(B, g.N, b_sn, b_sk, KB, KSB), false);
    if (bal || (guard && !staged)) {
      fusedA = !staged && kstats_lx(A, g.M, a_sm, a_sk, KA, KSA, EA);
      if (!fusedA) kstats(A, g.M, a_sm, a_sk, KA, KSA);
      have_ka = true;
    }
    balance_prep<<<1, 1024, 0, s>>>(KA, KB, bal ? g.K : 0, p.Kp, bal ? 1 : 0, SK, misc + 1);
    count();
    if (!staged) exponents(A, g.M, a_sm, a_sk, EA, +1, fusedA);
    exponents(B, g.N, b_sn, b_sk, EB, -1, fusedB);
    if (guard) {
      exp_max<<<1, 1024, 0, s>>>(EB, g.N, misc + 2);
      count();
    }
  }
  void res_args(ResArgs &r, bool isA, int64_t line0, int64_t lines_out, int8_t *out, int64_t plane_stride) const {
    r.base = isA ? g.A : g.B;
    r.nlines = isA ? g.M : g.N;
    r.K = g.K;
    r.Kp = p.Kp;
    r.s_l = isA ? a_sm : b_sn;
    r.s_k = isA ? a_sk : b_sk;
    r.line0 = line0;
    r.lines_out = lines_out;
    r.E = isA ? EA : EB;
    r.t = p.t;
    r.nmod = p.nmod;
    r.out = out;
    r.plane_stride = plane_stride;
    r.SK = SK;
    r.bal = misc + 1;
    r.sgn = isA ? 1 : -1;
    if (p.kind == kOzGauss) {
      // groups of the Gaussian moduli: 0-4, 5-9, 10-15 (products < 2^44)
      const int first[4] = {0, 5, 10, kMaxGMod};
      for (int gi = 0; gi < 3; gi++) {
        double P = 1.0;
        for (int l = first[gi]; l < std::min(first[gi + 1], p.nmod); l++) P *= (double)kGModuli[l];
        r.gP[gi] = P;                      // exact: < 2^44
        r.gPinv[gi] = 1.0 / P;
        r.gPlo[gi] = (int)(uint32_t)(uint64_t)P;
        r.gfirst[gi] = first[gi];
      }
      r.gfirst[3] = kMaxGMod;
    }
  }
  // after all chunks: guard, then the gated DMMA recomputation
  cudaError_t epilogue(bool cplx) {
    if (!guard) return cudaGetLastError();
    GuardArgs ga{};
    ga.EA = EA; ga.EB = EB; ga.M = g.M; ga.N = g.N; ga.K = g.K; ga.tpr = p.tpr;
    ga.KA = have_ka ? KA : nullptr; ga.KB = KB; ga.SK = SK;
    ga.KSA = have_ka ? KSA : nullptr; ga.KSB = KSB;
    ga.rowsq = rowsq; ga.t = p.t; ga.cplx = cplx ? 1 : 0; ga.tol = g.oz_tol;
    ga.flag = misc; ga.bal = misc + 1; ga.rec = g.oz_guard;
    if (p.tpr > 1) {   // fold each row's slots into its slot 0 first (many CTAs; fixed order)
      const unsigned blocks = (unsigned)std::min<int64_t>((g.M + 7) / 8, 4 * (int64_t)device_sms());
      rowsq_fold<<<blocks, 256, 0, s>>>(rowsq, g.M, p.tpr);
      count();
    }
    guard_finalize<<<1, 1024, 0, s>>>(ga);
    count();
    cudaError_t e = launch_gemm_dmma_if(g, misc, s, launches);
    if (e != cudaSuccess) return e;
    if (cplx && g.npeer > 0) {
      PeerSet ps{};
      for (int i = 0; i < g.npeer && i < 7; i++) ps.p[i] = static_cast<double2 *>(g.peer_C[i]);
      copy_to_peers_if<<<148 * 4, 256, 0, s>>>(static_cast<const double2 *>(g.C), g.M, g.N, g.c_sm,
                                                std::min(g.npeer, 7), ps, misc);
      count();
    }
    return cudaGetLastError();
  }
};

}  // namespace

// Load the guard's kernels now (CUDA lazy loading cannot load a kernel while
// a cross-rank barrier kernel of the same device spins: tci_gather_register)
cudaError_t ozaki_preload() {
  cudaFuncAttributes fa;
  const void *fns[] = {
      (const void *)copy_to_peers_if, (const void *)guard_finalize, (const void *)rowsq_fold, (const void *)exp_max,
      (const void *)balance_prep, (const void *)kstats_merge, (const void *)kstats_lines<double2>,
      (const void *)kstats_cols<double2>, (const void *)kstats_lines<double>, (const void *)kstats_cols<double>};
  if (cudaError_t e = crt_mma_preload(); e != cudaSuccess) return e;
  for (const void *f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

void ozaki_params(int64_t K, int kind, int *nmod, int *t, const int **moduli, const int **roots, int tmin) {
  const OzPlan p = oz_plan(1, 1, K, oz_budget(), 0, kind, tmin);
  if (nmod) *nmod = p.nmod;
  if (t) *t = p.t;
  if (moduli) *moduli = kind == kOzGauss ? kGModuli : kModuli;
  if (roots) *roots = kind == kOzGauss ? kGRoots : nullptr;
}

size_t ozaki_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  // sized for the largest plane count of any kind (3M, float64 sources) so
  // the variant can change without re-sizing
  return std::max(oz_plan(M, N, K, oz_budget(), 0, kOz3M).total,
                  oz_plan(M, N, K, oz_budget(), 0, kOzGauss).total);
}

namespace {

// C = A B (complex128, or complex64 with TS = TO = float2) per GemmProblem
// strides, by Ozaki-II on INT8 tcgen05.
template <class TS>
cudaError_t ozaki_zgemm_impl(const GemmProblem &g, void *ws, size_t ws_bytes, cudaStream_t s, int64_t *launches) {
  if (g.M == 0 || g.N == 0) return cudaSuccess;
  if (g.K > kOzakiMaxK) return cudaErrorInvalidValue;   // int32 residue products would overflow
  const bool gauss = g.oz_gauss != 0;
  const int tmin = std::is_same<TS, float2>::value ? kOzTminF32 : 46;
  const OzPlan p = oz_plan(g.M, g.N, g.K, oz_budget(), g.max_chunk_rows, gauss ? kOzGauss : kOz3M, tmin);
  if (ws_bytes < p.total || !ws) return cudaErrorInvalidValue;
  OzRun<TS> R(g, p, ws, s, launches);
  char *w = R.w;
  int8_t *Bres = reinterpret_cast<int8_t *>(w + p.off_Bres), *Ares = reinterpret_cast<int8_t *>(w + p.off_Ares);
  uint8_t *D = reinterpret_cast<uint8_t *>(w + p.off_D);
  R.prologue();
  const int planes = p.ppm * p.nmod;
  auto launch_res = [&](const ResArgs &r) {
    if (r.s_k == 1) {
      const unsigned blocks = (unsigned)((r.lines_out * (r.Kp / (gauss ? 4 : 8)) + 255) / 256);
      if (gauss)
        residues<true, TS><<<blocks, 256, 0, s>>>(r);
      else
        residues<false, TS><<<blocks, 256, 0, s>>>(r);
    } else {
      const unsigned blocks = (unsigned)(((r.lines_out + 31) / 32) * (r.Kp / 64));
      if (gauss)
        residues_t<true, TS><<<blocks, 256, 0, s>>>(r);
      else
        residues_t<false, TS><<<blocks, 256, 0, s>>>(r);
    }
    R.count();
  };
  {
    ResArgs r{};
    R.res_args(r, false, 0, p.Np, Bres, p.Np * p.Kp);
    launch_res(r);
  }
  CrtArgs c{};
  if (gauss) {
    crt_constants_gauss(p.nmod, c.W, c.WI, c.Mch, c.Minv);
  } else {
    double W[kMaxMod][4];
    crt_constants(p.nmod, W, c.Mch, c.Minv);
    for (int l = 0; l < kMaxMod; l++)
      for (int j = 0; j < 4; j++) c.W[l][j] = c.WI[l][j] = W[l][j];
  }
  {
    const double xs = gauss ? 512.0 : 1024.0;   // 2^XS of crt_kernel
    for (int j = 0; j < 4; j++) {
      double sr = 0.0, si = 0.0;
      for (int l = 0; l < p.nmod; l++) {
        sr += c.W[l][j];
        si += c.WI[l][j];
      }
      c.Cr[j] = xs * sr;
      c.Ci[j] = xs * si;
    }
  }
  c.nmod = p.nmod; c.EA = R.EA; c.EB = R.EB; c.t = p.t; c.N = g.N; c.Np = p.Np; c.D = D;
  c.C = g.C; c.c_sm = g.c_sm;
  c.npeer = std::min(g.npeer, 7);
  for (int pp = 0; pp < c.npeer; pp++) c.peer[pp] = g.peer_C[pp];
  c.rowsq = R.guard ? R.rowsq : nullptr;
  c.eb_max = R.misc + 2;
  using TO = TS;
  const bool crt_tc = gauss && crt_mma_enabled();
  CrtMmaArgs cm{};
  if (crt_tc) {
    crt_digits_gauss(p.nmod, cm);
    cm.D = D; cm.N = g.N; cm.Np = p.Np; cm.EA = R.EA; cm.EB = R.EB; cm.t = p.t;
    cm.C = g.C; cm.c_sm = g.c_sm; cm.npeer = c.npeer;
    for (int pp = 0; pp < c.npeer; pp++) cm.peer[pp] = c.peer[pp];
    cm.rowsq = c.rowsq; cm.slots_per_row = p.tpr; cm.eb_max = c.eb_max;
  }
  for (int64_t ch = 0; ch < p.chunks; ch++) {
    const int64_t m0 = ch * p.Mc, mc = std::min<int64_t>(p.Mc, g.M - m0);
    if (g.rows_needed) {
      g.rows_needed(g.rows_user, m0, mc);
      R.exponents(static_cast<const TS *>(g.A) + m0 * g.a_sm, mc, g.a_sm, g.a_sk, R.EA + m0, +1);
    }
    {
      ResArgs r{};
      R.res_args(r, true, m0, mc, Ares, mc * p.Kp);
      launch_res(r);
    }
    cudaError_t ge = int8_gemm(g, p, Ares, Bres, D, mc, planes, p.ppm, R.misc + 3, s, launches);
    if (ge != cudaSuccess) return ge;
    c.Mc = mc;
    c.m0 = m0;
    cudaError_t ce;
    if (crt_tc) {
      cm.Mc = mc;
      cm.m0 = m0;
      ce = launch_crt_mma(cm, std::is_same<TO, float2>::value, false, s);
    } else if (gauss) {
      switch (p.nmod) {
        case 9: ce = launch_crt<9, 2, true, TO>(c, mc, s); break;
        case 10: ce = launch_crt<10, 2, true, TO>(c, mc, s); break;
        case 11: ce = launch_crt<11, 3, true, TO>(c, mc, s); break;
        case 15: ce = launch_crt<15, 3, true, TO>(c, mc, s); break;
        case 16: ce = launch_crt<16, 4, true, TO>(c, mc, s); break;
        default: return cudaErrorInvalidValue;
      }
    } else {
      switch (p.nmod) {
        case 8: ce = launch_crt<8, 2, false, TO>(c, mc, s); break;
        case 9: ce = launch_crt<9, 2, false, TO>(c, mc, s); break;
        case 10: ce = launch_crt<10, 3, false, TO>(c, mc, s); break;
        case 12: ce = launch_crt<12, 3, false, TO>(c, mc, s); break;
        case 13: ce = launch_crt<13, 3, false, TO>(c, mc, s); break;
        case 14: ce = launch_crt<14, 3, false, TO>(c, mc, s); break;
        case 15: ce = launch_crt<15, 4, false, TO>(c, mc, s); break;
        default: return cudaErrorInvalidValue;
      }
    }
    if (ce != cudaSuccess) return ce;
    R.count();
    if (g.rows_done) g.rows_done(g.rows_user, m0, mc);
  }
  return R.epilogue(true);
}

// C = A B (float64, or float32 with TS = float) by real Ozaki-II on INT8
// tcgen05 (layout of ozaki_workspace_bytes: sized for 3n planes, n used here).
template <class TS>
cudaError_t ozaki_dgemm_impl(const GemmProblem &g, void *ws, size_t ws_bytes, cudaStream_t s, int64_t *launches) {
  if (g.M == 0 || g.N == 0) return cudaSuccess;
  if (g.K > kOzakiMaxK) return cudaErrorInvalidValue;
  if (g.rows_needed) return cudaErrorInvalidValue;   // the real path takes all row exponents up front
  const int tmin = std::is_same<TS, float>::value ? kOzTminF32 : 46;
  const OzPlan p = oz_plan(g.M, g.N, g.K, oz_budget(), g.max_chunk_rows, kOzReal, tmin);
  if (ws_bytes < p.total || !ws) return cudaErrorInvalidValue;
  OzRun<TS> R(g, p, ws, s, launches);
  char *w = R.w;
  int8_t *Bres = reinterpret_cast<int8_t *>(w + p.off_Bres), *Ares = reinterpret_cast<int8_t *>(w + p.off_Ares);
  uint8_t *D = reinterpret_cast<uint8_t *>(w + p.off_D);
  R.prologue();
  auto launch_res = [&](const ResArgs &r) {
    if (r.s_k == 1) {
      const int64_t th = r.lines_out * (r.Kp / 8);
      residues_real<TS><<<(unsigned)((th + 255) / 256), 256, 0, s>>>(r);
    } else {
      residues_real_t<TS><<<(unsigned)(((r.lines_out + 31) / 32) * (r.Kp / 64)), 256, 0, s>>>(r);
    }
    R.count();
  };
  const int planes = p.nmod;
  {
    ResArgs r{};
    R.res_args(r, false, 0, p.Np, Bres, p.Np * p.Kp);
    launch_res(r);
  }
  CrtArgsR c{};
  crt_constants(p.nmod, c.W, c.Mch, c.Minv);
  for (int j = 0; j < 4; j++) {
    double sw = 0.0;
    for (int l = 0; l < p.nmod; l++) sw += c.W[l][j];
    c.C0[j] = 256.0 * sw;
  }
  c.nmod = p.nmod; c.EA = R.EA; c.EB = R.EB; c.t = p.t; c.N = g.N; c.Np = p.Np; c.D = D;
  c.C = g.C; c.c_sm = g.c_sm;
  c.rowsq = R.guard ? R.rowsq : nullptr;
  c.eb_max = R.misc + 2;
  using TO = TS;
  const bool crt_tc = crt_mma_enabled();
  CrtMmaArgs cm{};
  if (crt_tc) {
    crt_digits_real(p.nmod, cm);
    cm.D = D; cm.N = g.N; cm.Np = p.Np; cm.EA = R.EA; cm.EB = R.EB; cm.t = p.t;
    cm.C = g.C; cm.c_sm = g.c_sm; cm.npeer = 0;
    cm.rowsq = c.rowsq; cm.slots_per_row = p.tpr; cm.eb_max = c.eb_max;
  }
  for (int64_t ch = 0; ch < p.chunks; ch++) {
    const int64_t m0 = ch * p.Mc, mc = std::min<int64_t>(p.Mc, g.M - m0);
    {
      ResArgs r{};
      R.res_args(r, true, m0, mc, Ares, mc * p.Kp);
      launch_res(r);
    }
    cudaError_t ge = int8_gemm(g, p, Ares, Bres, D, mc, planes, 1, R.misc + 3, s, launches);
    if (ge != cudaSuccess) return ge;
    c.Mc = mc;
    c.m0 = m0;
    if (crt_tc) {   // the tensor-core CRT (crt_mma.cu), real outputs
      cm.Mc = mc;
      cm.m0 = m0;
      cudaError_t ce = launch_crt_mma(cm, std::is_same<TO, float>::value, true, s);
      if (ce != cudaSuccess) return ce;
      R.count();
      if (g.rows_done) g.rows_done(g.rows_user, m0, mc);
      continue;
    }
    const unsigned blocks = (unsigned)(mc * p.tpr);
    switch (p.nmod) {
      case 8: crt_real_kernel<8, 2, TO><<<blocks, 256, 0, s>>>(c); break;
      case 9: crt_real_kernel<9, 2, TO><<<blocks, 256, 0, s>>>(c); break;
      case 10: crt_real_kernel<10, 3, TO><<<blocks, 256, 0, s>>>(c); break;
      case 12: crt_real_kernel<12, 3, TO><<<blocks, 256, 0, s>>>(c); break;
      case 13: crt_real_kernel<13, 3, TO><<<blocks, 256, 0, s>>>(c); break;
      case 14: crt_real_kernel<14, 3, TO><<<blocks, 256, 0, s>>>(c); break;
      case 15: crt_real_kernel<15, 4, TO><<<blocks, 256, 0, s>>>(c); break;
      default: return cudaErrorInvalidValue;
    }
    R.count();
    if (g.rows_done) g.rows_done(g.rows_user, m0, mc);
  }
  return R.epilogue(false);
}

}  // namespace

cudaError_t launch_ozaki_zgemm(const GemmProblem &g, void *ws, size_t ws_bytes, cudaStream_t s,
                               int64_t *launches) {
  return g.dtype == TCI_C64 ? ozaki_zgemm_impl<float2>(g, ws, ws_bytes, s, launches)
                            : ozaki_zgemm_impl<double2>(g, ws, ws_bytes, s, launches);
}

cudaError_t launch_ozaki_dgemm(const GemmProblem &g, void *ws, size_t ws_bytes, cudaStream_t s,
                               int64_t *launches) {
  return g.dtype == TCI_R32 ? ozaki_dgemm_impl<float>(g, ws, ws_bytes, s, launches)
                            : ozaki_dgemm_impl<double>(g, ws, ws_bytes, s, launches);
}

}  // namespace tci
