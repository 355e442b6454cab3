// skinny.cu -- small-K / small-N contraction (SURVEY 8(a5) MPO passes,
// 8(a10) site-local MPS-MPO application, TEBD gate pass):
//   out[b0,b1,b2, n] = sum_{k < K} in[b0,b1,b2, k] * W(k, n),  K, N <= 128
// with arbitrary strides on every leg (offset tables for the fused k and n
// groups, passed by value). These contractions move each element once for a
// few tens of MACs, so they are HBM-bound (or near the HBM/FP64 balance for
// the fused W12 pass at d=2): a tensor-core GEMM tile would idle on K=4..96,
// so this is a CUDA-core kernel whose job is to stream `in` and `out` once
// with coalesced accesses.
//
// One CTA owns TB consecutive values of the fastest batch leg b2 for one
// (b0,b1): it stages the [K x TB] input tile and W in shared memory, each
// thread accumulates a slice of the N outputs of one b2 value (k ascending,
// fixed order -> deterministic), and results are staged in shared memory and
// written back in (n_hi, b2, n_lo) order so global stores are contiguous when
// the trailing n-run is interleaved with b2.
#include <algorithm>
#include <cstdlib>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

template <bool CPLX>
struct SkE;
template <>
struct SkE<false> {
  using T = double;
  static __device__ __forceinline__ T zero() { return 0.0; }
  static __device__ __forceinline__ void mac(T &c, T a, T b) { c = fma(a, b, c); }
};
template <>
struct SkE<true> {
  using T = double2;
  static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ void mac(T &c, T a, T b) {
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(-a.y, b.y, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.y = fma(a.y, b.x, c.y);
  }
};

constexpr int TB = 64;        // b2 values per CTA
constexpr int NTH = 256;      // threads
constexpr int NG = NTH / TB;  // n-groups per b2 value
constexpr int MAXNPT = kSkinnyMaxN / NG;

template <bool CPLX, int NPT>
__global__ void __launch_bounds__(NTH) skinny_kernel(const __grid_constant__ SkinnyProblem a) {
  using Ops = SkE<CPLX>;
  using T = typename Ops::T;
  extern __shared__ __align__(16) char sm[];
  const int K = a.K, N = a.N;
  T *sW = reinterpret_cast<T *>(sm);   // [K][N]
  T *sIn = sW + K * N;                 // [K][TB]
  T *sOut = sIn + K * TB;              // [TB][N]

  const int64_t tiles2 = (a.nb[2] + TB - 1) / TB;
  int64_t bid = blockIdx.x;
  const int64_t t2 = bid % tiles2;
  bid /= tiles2;
  const int64_t i1 = bid % a.nb[1];
  const int64_t i0 = bid / a.nb[1];
  const int64_t c0 = t2 * TB;
  const int nc = (int)min((int64_t)TB, a.nb[2] - c0);
  const T *in = reinterpret_cast<const T *>(a.in) + i0 * a.in_sb[0] + i1 * a.in_sb[1] + c0 * a.in_sb[2];
  T *out = reinterpret_cast<T *>(a.out) + i0 * a.out_sb[0] + i1 * a.out_sb[1] + c0 * a.out_sb[2];
  const T *W = reinterpret_cast<const T *>(a.W);
  const int tid = threadIdx.x;

  for (int i = tid; i < K * N; i += NTH) {
    const int k = i / N, n = i % N;
    sW[i] = W[a.w_koff[k] + a.w_noff[n]];
  }
  // load: (k_hi, c, k_lo) order -> contiguous reads when in_sb[2] == k_lo
  for (int idx = tid; idx < K * TB; idx += NTH) {
    const int khi = idx / (TB * a.k_lo), rem = idx % (TB * a.k_lo);
    const int c = rem / a.k_lo, k = khi * a.k_lo + rem % a.k_lo;
    sIn[k * TB + c] = (c < nc) ? in[c * a.in_sb[2] + a.in_koff[k]] : Ops::zero();
  }
  __syncthreads();
  {
    const int c = tid % TB, g = tid / TB;
    T acc[NPT];
#pragma unroll
    for (int j = 0; j < NPT; j++) acc[j] = Ops::zero();
    for (int k = 0; k < K; k++) {
      const T x = sIn[k * TB + c];
#pragma unroll
      for (int j = 0; j < NPT; j++) {
        const int n = g + j * NG;
        if (n < N) Ops::mac(acc[j], x, sW[k * N + n]);
      }
    }
#pragma unroll
    for (int j = 0; j < NPT; j++) {
      const int n = g + j * NG;
      if (n < N) sOut[c * N + n] = acc[j];
    }
  }
  __syncthreads();
  // store: (n_hi, c, n_lo) order
  for (int idx = tid; idx < N * TB; idx += NTH) {
    const int nhi = idx / (TB * a.n_lo), rem = idx % (TB * a.n_lo);
    const int c = rem / a.n_lo, n = nhi * a.n_lo + rem % a.n_lo;
    if (c < nc) out[c * a.out_sb[2] + a.out_noff[n]] = sOut[c * N + n];
  }
}

// ---------------------------------------------------------------------------
// Streaming variant (b2 contiguous in the input, k_lo == 1): persistent CTAs,
// the [K x TB] input tile of the next (b0, b1, b2-block) is prefetched with
// cp.async while the current one is contracted; each thread owns NPT
// CONSECUTIVE outputs n = g*NPT .. g*NPT + NPT - 1 of one b2 value and stores
// them straight from registers (with the trailing n-run interleaved with b2,
// as in the H_eff MPO pass, a warp then writes one contiguous block).
// Complex products use 3 real multiplications (Gauss / 3M, as the DMMA GEMM):
// P = sum xr wr, Q = sum xi wi, S = sum (xr + xi)(wr + wi); re = P - Q,
// im = S - P - Q (normwise stable, R11).
// ---------------------------------------------------------------------------
constexpr int NC = 2;            // b2 values per thread (register blocking: weights reused NC times)
constexpr int TBS = TB * NC;     // b2 values per streamed tile

template <bool CPLX, int NPT, bool FULL>
__global__ void __launch_bounds__(NTH) skinny_stream_kernel(const __grid_constant__ SkinnyProblem a,
                                                            int64_t ntiles) {
  using T = typename SkE<CPLX>::T;
  constexpr int NW = CPLX ? 3 : 1;       // weight planes: (wr, wi, wr + wi) or w
  extern __shared__ __align__(16) char sm[];
  const int K = a.K, N = a.N;
  double *sW = reinterpret_cast<double *>(sm);                    // [NW][K][N]
  T *sIn = reinterpret_cast<T *>(sW + NW * K * N + (NW * K * N) % 2);   // [2][K][TBS], 16 B aligned
  const T *W = reinterpret_cast<const T *>(a.W);
  const int tid = threadIdx.x;
  for (int i = tid; i < K * N; i += NTH) {
    const int k = i / N, n = i % N;
    const T w = W[a.w_koff[k] + a.w_noff[n]];
    if constexpr (CPLX) {
      sW[i] = w.x;
      sW[K * N + i] = w.y;
      sW[2 * K * N + i] = w.x + w.y;
    } else {
      sW[i] = w;
    }
  }
  const int64_t tiles2 = (a.nb[2] + TBS - 1) / TBS;
  auto tile_ptrs = [&](int64_t t, const T *&in, T *&out, int &nc) {
    const int64_t t2 = t % tiles2, r = t / tiles2;
    const int64_t i1 = r % a.nb[1], i0 = r / a.nb[1];
    const int64_t c0 = t2 * TBS;
    nc = (int)min((int64_t)TBS, a.nb[2] - c0);
    in = reinterpret_cast<const T *>(a.in) + i0 * a.in_sb[0] + i1 * a.in_sb[1] + c0;
    out = reinterpret_cast<T *>(a.out) + i0 * a.out_sb[0] + i1 * a.out_sb[1] + c0 * a.out_sb[2];
  };
  constexpr int PER16 = 16 / (int)sizeof(T);   // elements per 16-byte copy
  auto load = [&](int64_t t, int buf) {
    const T *in;
    T *out;
    int nc;
    tile_ptrs(t, in, out, nc);
    T *dst = sIn + buf * K * TBS;
    constexpr int CPR = TBS / PER16;
    for (int i = tid; i < K * CPR; i += NTH) {
      const int k = i / CPR, q = i % CPR;
      const int c = q * PER16;
      const int valid = c < nc ? (int)min(16, (nc - c) * (int)sizeof(T)) : 0;
      cp_async_zfill<16>(dst + k * TBS + c, valid ? in + a.in_koff[k] + c : in, valid);
    }
  };
  int64_t t = blockIdx.x;
  if (t < ntiles) load(t, 0);
  cp_async_commit();
  const int cl = tid % TB, g = tid / TB;   // b2 values cl + TB * i, outputs g*NPT ..
  const int n0 = g * NPT;
  int buf = 0;
  for (; t < ntiles; t += gridDim.x, buf ^= 1) {
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) load(tn, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const T *tile = sIn + buf * K * TBS;
    const T *in;
    T *out;
    int nc;
    tile_ptrs(t, in, out, nc);
    if constexpr (CPLX) {
      double P[NC][NPT], Q[NC][NPT], S[NC][NPT];
#pragma unroll
      for (int i = 0; i < NC; i++)
#pragma unroll
        for (int j = 0; j < NPT; j++) P[i][j] = Q[i][j] = S[i][j] = 0.0;
#pragma unroll 2
      for (int k = 0; k < K; k++) {
        double xr[NC], xi[NC], xs[NC];
#pragma unroll
        for (int i = 0; i < NC; i++) {
          const T x = tile[k * TBS + cl + TB * i];
          xr[i] = x.x;
          xi[i] = x.y;
          xs[i] = x.x + x.y;
        }
        const double *wr = sW + k * N + n0, *wi = wr + K * N, *ws = wi + K * N;
#pragma unroll
        for (int j = 0; j < NPT; j++) {
          if (FULL || n0 + j < N) {
            const double a_ = wr[j], b_ = wi[j], c_ = ws[j];
#pragma unroll
            for (int i = 0; i < NC; i++) {
              P[i][j] = fma(xr[i], a_, P[i][j]);
              Q[i][j] = fma(xi[i], b_, Q[i][j]);
              S[i][j] = fma(xs[i], c_, S[i][j]);
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NC; i++) {
        const int c = cl + TB * i;
        if (c < nc) {
#pragma unroll
          for (int j = 0; j < NPT; j++)
            if (FULL || n0 + j < N)
              out[c * a.out_sb[2] + a.out_noff[n0 + j]] =
                  make_double2(P[i][j] - Q[i][j], S[i][j] - P[i][j] - Q[i][j]);
        }
      }
    } else {
      double acc[NC][NPT];
#pragma unroll
      for (int i = 0; i < NC; i++)
#pragma unroll
        for (int j = 0; j < NPT; j++) acc[i][j] = 0.0;
#pragma unroll 2
      for (int k = 0; k < K; k++) {
        double x[NC];
#pragma unroll
        for (int i = 0; i < NC; i++) x[i] = tile[k * TBS + cl + TB * i];
        const double *w = sW + k * N + n0;
#pragma unroll
        for (int j = 0; j < NPT; j++)
          if (FULL || n0 + j < N) {
            const double wj = w[j];
#pragma unroll
            for (int i = 0; i < NC; i++) acc[i][j] = fma(x[i], wj, acc[i][j]);
          }
      }
#pragma unroll
      for (int i = 0; i < NC; i++) {
        const int c = cl + TB * i;
        if (c < nc) {
#pragma unroll
          for (int j = 0; j < NPT; j++)
            if (FULL || n0 + j < N) out[c * a.out_sb[2] + a.out_noff[n0 + j]] = acc[i][j];
        }
      }
    }
    __syncthreads();   // this buffer is refilled two tiles later
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Expansion variant (K <= 8, N >= 4 K: output-write bound, e.g. the site-local
// MPS-MPO application B[a,w,t,b,v] = sum_s A[a,s,b] W[w,v,s,t], 8(a10)): when
// the trailing n-run of length n_lo sits right after b2 in the output
// (out_sb[2] == n_lo, each run contiguous), the outputs of a tile of TBX b2
// values form, for every leading n-group, ONE contiguous block of TBX n_lo
// elements. Each thread computes the elements it stores -- consecutive
// lanes, consecutive addresses -- straight from the staged input tile and W
// (shared memory), so every warp store is a contiguous 512-byte run (complex)
// and nothing is staged on the way out. Persistent CTAs, several per SM, hide
// the per-tile input latency. Complex products are direct (4 real FMAs per
// MAC, k ascending): exact for unit / zero weights.
// ---------------------------------------------------------------------------
constexpr int TBX = 128;          // b2 values per tile
constexpr int kExpandMaxK = 8, kExpandMaxNL = 8;
constexpr int kExpandJ = TBX * kExpandMaxNL / NTH;   // block elements per thread (<= 4)

template <bool CPLX>
__global__ void __launch_bounds__(NTH) skinny_expand_kernel(const __grid_constant__ SkinnyProblem a,
                                                            int64_t ntiles) {
  using Ops = SkE<CPLX>;
  using T = typename Ops::T;
  extern __shared__ __align__(16) char sm[];
  const int K = a.K, N = a.N, NL = a.n_lo, NH = N / NL;
  T *sW = reinterpret_cast<T *>(sm);   // [K][N]
  T *sIn = sW + K * N;                 // [K][TBX]
  const T *W = reinterpret_cast<const T *>(a.W);
  const int tid = threadIdx.x;
  for (int i = tid; i < K * N; i += NTH) {
    const int k = i / N, n = i % N;
    sW[i] = W[a.w_koff[k] + a.w_noff[n]];
  }
  // this thread's block elements i = tid + NTH j -> (b2 offset c, run position l): fixed for every tile
  int cc[kExpandJ], ll[kExpandJ];
#pragma unroll
  for (int j = 0; j < kExpandJ; j++) {
    const int i = tid + NTH * j;
    cc[j] = i / NL;
    ll[j] = i % NL;
  }
  const int64_t tiles2 = (a.nb[2] + TBX - 1) / TBX;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t t2 = t % tiles2, r = t / tiles2;
    const int64_t i1 = r % a.nb[1], i0 = r / a.nb[1];
    const int64_t c0 = t2 * TBX;
    const int nc = (int)min((int64_t)TBX, a.nb[2] - c0);
    const T *in = reinterpret_cast<const T *>(a.in) + i0 * a.in_sb[0] + i1 * a.in_sb[1] + c0 * a.in_sb[2];
    T *out = reinterpret_cast<T *>(a.out) + i0 * a.out_sb[0] + i1 * a.out_sb[1] + c0 * a.out_sb[2];
    __syncthreads();   // the previous tile is done with sIn
    for (int i = tid; i < K * TBX; i += NTH) {
      const int k = i / TBX, c = i % TBX;
      sIn[i] = c < nc ? in[c * a.in_sb[2] + a.in_koff[k]] : Ops::zero();
    }
    __syncthreads();
    const int nb = nc * NL;   // valid elements of each block
    for (int nh = 0; nh < NH; nh++) {
      T *ob = out + a.out_noff[nh * NL];
      const T *w = sW + nh * NL;
#pragma unroll
      for (int j = 0; j < kExpandJ; j++) {
        const int i = tid + NTH * j;
        if (i < nb) {
          T acc = Ops::zero();
          for (int k = 0; k < K; k++) Ops::mac(acc, sIn[k * TBX + cc[j]], w[k * N + ll[j]]);
          __stcs(ob + i, acc);
        }
      }
    }
  }
}

template <bool CPLX>
cudaError_t launch_expand(const SkinnyProblem &p, cudaStream_t s) {
  const size_t es = CPLX ? 16 : 8;
  const size_t smem = (size_t)(p.K * p.N + p.K * TBX) * es;
  const int64_t ntiles = p.nb[0] * p.nb[1] * ((p.nb[2] + TBX - 1) / TBX);
  auto k = skinny_expand_kernel<CPLX>;
  cudaError_t e = ensure_smem_attr((const void *)k, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = occupancy_per_sm((const void *)k, NTH, smem);
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)device_sms() * std::max(1, per_sm));
  k<<<(unsigned)grid, NTH, smem, s>>>(p, ntiles);
  return cudaGetLastError();
}

// the expansion layout: few k, many n, the n-runs of length n_lo contiguous
// and interleaved right after b2 in the output
bool expand_ok(const SkinnyProblem &p) {
  if (p.K > kExpandMaxK || p.N < 4 * p.K || p.n_lo < 1 || p.n_lo > kExpandMaxNL || p.N % p.n_lo) return false;
  if (p.out_sb[2] != p.n_lo || p.nb[2] < TBX / 2) return false;
  for (int n = 0; n < p.N; n++)
    if (p.out_noff[n] != p.out_noff[n - n % p.n_lo] + n % p.n_lo) return false;
  const size_t es = p.dtype == TCI_C128 ? 16 : 8;
  return (uintptr_t)p.out % es == 0;
}

// ---------------------------------------------------------------------------
// Tensor-core variant of the streaming complex pass (K, N <= 32; the H_eff
// MPO pass is K = N = 20 at d = 2, D = 5): the contraction of a tile of TD
// b2 values is the [TD x K] x [K x N] product, run as FP64 DMMA m8n8k4 with
// the 3M complex split (P = Xr Wr, Q = Xi Wi, S = (Xr + Xi)(Wr + Wi); re =
// P - Q, im = S - P - Q, as the streaming CUDA-core kernel). One DMMA does
// 256 FMAs, so the pass needs ~1/8 of the FP64 instructions of the CUDA-core
// version and is left bound by streaming `in` and `out` (HBM). W's three
// planes sit in shared memory pre-arranged as per-lane B fragments; the input
// tile [K][TD] is double-buffered with cp.async; warp w owns m-tile w (8 b2
// values). Summation order per output: k ascending in chunks of 4 (DMMA),
// fixed -> deterministic.
// ---------------------------------------------------------------------------
template <int KS, int NTL, int MT>
__global__ void __launch_bounds__(NTH) skinny_dmma_kernel(const __grid_constant__ SkinnyProblem a, int64_t ntiles) {
  constexpr int TD = 8 * (NTH / 32) * MT;   // b2 values per tile: MT m-tiles of 8 per warp
  extern __shared__ __align__(16) char sm[];
  const int K = a.K, N = a.N;
  double *sWf = reinterpret_cast<double *>(sm);                        // [KS][NTL][3][32]
  const int KN = K > N ? K : N;                                        // buffer rows: input [K] / output [N]
  double2 *sIn = reinterpret_cast<double2 *>(sWf + KS * NTL * 3 * 32);  // [2][KN][TD]
  const double2 *W = reinterpret_cast<const double2 *>(a.W);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int wimag = 0;
  for (int i = tid; i < KS * NTL * 32; i += NTH) {
    const int l = i & 31, f = i >> 5, nt = f % NTL, ks = f / NTL;
    const int k = ks * 4 + (l & 3), n = nt * 8 + (l >> 2);
    double2 w = make_double2(0.0, 0.0);
    if (k < K && n < N) w = W[a.w_koff[k] + a.w_noff[n]];
    double *dst = sWf + ((ks * NTL + nt) * 3) * 32 + l;
    dst[0] = w.x;
    dst[32] = w.y;
    dst[64] = w.x + w.y;
    wimag |= (w.y != 0.0);
  }
  // a real W (the Heisenberg / Hubbard MPOs): X W = (Xr W, Xi W), two DMMAs
  // per fragment product instead of the three of 3M (uniform per CTA)
  const bool wreal = __syncthreads_or(wimag) == 0;
  const int64_t tiles2 = (a.nb[2] + TD - 1) / TD;
  auto tile_ptrs = [&](int64_t t, const double2 *&in, double2 *&out, int &nc) {
    const int64_t t2 = t % tiles2, r = t / tiles2;
    const int64_t i1 = r % a.nb[1], i0 = r / a.nb[1];
    const int64_t c0 = t2 * TD;
    nc = (int)min((int64_t)TD, a.nb[2] - c0);
    in = reinterpret_cast<const double2 *>(a.in) + i0 * a.in_sb[0] + i1 * a.in_sb[1] + c0;
    out = reinterpret_cast<double2 *>(a.out) + i0 * a.out_sb[0] + i1 * a.out_sb[1] + c0 * a.out_sb[2];
  };
  auto load = [&](int64_t t, int buf) {
    const double2 *in;
    double2 *out;
    int nc;
    tile_ptrs(t, in, out, nc);
    double2 *dst = sIn + buf * KN * TD;
    for (int i = tid; i < K * TD; i += NTH) {
      const int k = i / TD, c = i % TD;
      cp_async_zfill<16>(dst + k * TD + c, c < nc ? in + a.in_koff[k] + c : in, c < nc ? 16 : 0);
    }
  };
  int64_t t = blockIdx.x;
  if (t < ntiles) load(t, 0);
  cp_async_commit();
  int buf = 0;
  const int r = lane >> 2, q = lane & 3;   // fragment row (b2 in the m-tile) / column (k in the step)
  for (; t < ntiles; t += gridDim.x, buf ^= 1) {
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) load(tn, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double2 *tile = sIn + buf * KN * TD;
    const double2 *in;
    double2 *out;
    int nc;
    tile_ptrs(t, in, out, nc);
    double P[MT][NTL][2], Q[MT][NTL][2], S[MT][NTL][2];
#pragma unroll
    for (int m = 0; m < MT; m++)
#pragma unroll
      for (int nt = 0; nt < NTL; nt++)
#pragma unroll
        for (int e = 0; e < 2; e++) P[m][nt][e] = Q[m][nt][e] = S[m][nt][e] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ks++) {
      const int k = ks * 4 + q;
      double ar[MT], ai[MT], as[MT];
#pragma unroll
      for (int m = 0; m < MT; m++) {
        const double2 x = k < K ? tile[k * TD + (warp * MT + m) * 8 + r] : make_double2(0.0, 0.0);
        ar[m] = x.x;
        ai[m] = x.y;
        as[m] = x.x + x.y;
      }
      if (wreal) {
#pragma unroll
        for (int nt = 0; nt < NTL; nt++) {
          const double wr = sWf[((ks * NTL + nt) * 3) * 32 + lane];
#pragma unroll
          for (int m = 0; m < MT; m++) {
            dmma884(P[m][nt], ar[m], wr);
            dmma884(Q[m][nt], ai[m], wr);
          }
        }
      } else {
#pragma unroll
        for (int nt = 0; nt < NTL; nt++) {
          const double *wf = sWf + ((ks * NTL + nt) * 3) * 32 + lane;
          const double wr = wf[0], wi = wf[32], ws = wf[64];
#pragma unroll
          for (int m = 0; m < MT; m++) {
            dmma884(P[m][nt], ar[m], wr);
            dmma884(Q[m][nt], ai[m], wi);
            dmma884(S[m][nt], as[m], ws);
          }
        }
      }
    }
    // C fragment: row r (b2), columns n = nt*8 + 2q + e, stored from registers
    // (staging through shared memory for contiguous warp stores measured slower:
    // 2.92 vs 2.60 ms at the target, the extra barriers cost more than L2 merging)
#pragma unroll
    for (int m = 0; m < MT; m++) {
      const int c = (warp * MT + m) * 8 + r;
      if (c < nc) {
#pragma unroll
        for (int nt = 0; nt < NTL; nt++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int n = nt * 8 + 2 * q + e;
            if (n < N)
              out[c * a.out_sb[2] + a.out_noff[n]] =
                  wreal ? make_double2(P[m][nt][e], Q[m][nt][e])
                        : make_double2(P[m][nt][e] - Q[m][nt][e], S[m][nt][e] - P[m][nt][e] - Q[m][nt][e]);
          }
      }
    }
    __syncthreads();   // this buffer is refilled two tiles later
  }
  cp_async_wait<0>();
}

template <int KS, int NTL, int MT>
cudaError_t launch_dmma_knm(const SkinnyProblem &p, cudaStream_t s) {
  constexpr int TD = 8 * (NTH / 32) * MT;
  const size_t smem = (size_t)KS * NTL * 3 * 32 * 8 + 2 * (size_t)std::max(p.K, p.N) * TD * 16;
  const int64_t ntiles = p.nb[0] * p.nb[1] * ((p.nb[2] + TD - 1) / TD);
  auto k = skinny_dmma_kernel<KS, NTL, MT>;
  cudaError_t e = ensure_smem_attr((const void *)k, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = occupancy_per_sm((const void *)k, NTH, smem);
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)148 * std::max(1, per_sm));
  k<<<(unsigned)grid, NTH, smem, s>>>(p, ntiles);
  return cudaGetLastError();
}

template <int KS, int NTL>
cudaError_t launch_dmma_kn(const SkinnyProblem &p, cudaStream_t s) {
  return launch_dmma_knm<KS, NTL, 1>(p, s);   // one m-tile per warp: 2.60 ms vs 2.70 (two) at the target
}

template <int KS>
cudaError_t launch_dmma_k(const SkinnyProblem &p, cudaStream_t s) {
  switch ((p.N + 7) / 8) {
    case 1: return launch_dmma_kn<KS, 1>(p, s);
    case 2: return launch_dmma_kn<KS, 2>(p, s);
    case 3: return launch_dmma_kn<KS, 3>(p, s);
    default: return launch_dmma_kn<KS, 4>(p, s);
  }
}

// K, N <= 32, complex, b2 unit-stride in the input (the caller checked)
cudaError_t launch_dmma(const SkinnyProblem &p, cudaStream_t s) {
  switch ((p.K + 3) / 4) {
    case 1: return launch_dmma_k<1>(p, s);
    case 2: return launch_dmma_k<2>(p, s);
    case 3: return launch_dmma_k<3>(p, s);
    case 4: return launch_dmma_k<4>(p, s);
    case 5: return launch_dmma_k<5>(p, s);
    case 6: return launch_dmma_k<6>(p, s);
    case 7: return launch_dmma_k<7>(p, s);
    default: return launch_dmma_k<8>(p, s);
  }
}

template <bool CPLX, int NPT>
cudaError_t launch_stream_npt(const SkinnyProblem &p, cudaStream_t s) {
  const size_t es = CPLX ? 16 : 8;
  const int NW = CPLX ? 3 : 1;
  const size_t smem = (size_t)(NW * p.K * p.N + (NW * p.K * p.N) % 2) * 8 + 2 * (size_t)p.K * TBS * es;
  const int64_t ntiles = p.nb[0] * p.nb[1] * ((p.nb[2] + TBS - 1) / TBS);
  auto k = (p.N == NPT * NG) ? skinny_stream_kernel<CPLX, NPT, true> : skinny_stream_kernel<CPLX, NPT, false>;
  cudaError_t e = ensure_smem_attr((const void *)k, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = occupancy_per_sm((const void *)k, NTH, smem);
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)148 * std::max(1, per_sm));
  k<<<(unsigned)grid, NTH, smem, s>>>(p, ntiles);
  return cudaGetLastError();
}

template <bool CPLX>
cudaError_t launch_stream(const SkinnyProblem &p, cudaStream_t s) {
  const int npt = (p.N + NG - 1) / NG;
  switch (npt) {
    case 1: return launch_stream_npt<CPLX, 1>(p, s);
    case 2: return launch_stream_npt<CPLX, 2>(p, s);
    case 3: return launch_stream_npt<CPLX, 3>(p, s);
    case 4: return launch_stream_npt<CPLX, 4>(p, s);
    case 5: return launch_stream_npt<CPLX, 5>(p, s);
    case 6: return launch_stream_npt<CPLX, 6>(p, s);
  }
  if (npt <= 8) return launch_stream_npt<CPLX, 8>(p, s);
  if (npt <= 12) return launch_stream_npt<CPLX, 12>(p, s);
  if (npt <= 16) return launch_stream_npt<CPLX, 16>(p, s);
  return launch_stream_npt<CPLX, MAXNPT>(p, s);
}

template <bool CPLX, int NPT>
cudaError_t launch_npt(const SkinnyProblem &p, size_t smem, int64_t blocks, cudaStream_t s) {
  auto k = skinny_kernel<CPLX, NPT>;
  cudaError_t e = ensure_smem_attr((const void *)k, smem);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)blocks, NTH, smem, s>>>(p);
  return cudaGetLastError();
}

template <bool CPLX>
cudaError_t launch_c(const SkinnyProblem &p, size_t smem, int64_t blocks, cudaStream_t s) {
  // outputs per thread: instantiated exactly for the common sizes so no
  // unrolled slot is dead (N = 20 -> 5 at d=2, D=5)
  const int npt = (p.N + NG - 1) / NG;
  switch (npt) {
    case 1: return launch_npt<CPLX, 1>(p, smem, blocks, s);
    case 2: return launch_npt<CPLX, 2>(p, smem, blocks, s);
    case 3: return launch_npt<CPLX, 3>(p, smem, blocks, s);
    case 4: return launch_npt<CPLX, 4>(p, smem, blocks, s);
    case 5: return launch_npt<CPLX, 5>(p, smem, blocks, s);
    case 6: return launch_npt<CPLX, 6>(p, smem, blocks, s);
  }
  if (npt <= 8) return launch_npt<CPLX, 8>(p, smem, blocks, s);
  if (npt <= 12) return launch_npt<CPLX, 12>(p, smem, blocks, s);
  if (npt <= 16) return launch_npt<CPLX, 16>(p, smem, blocks, s);
  return launch_npt<CPLX, MAXNPT>(p, smem, blocks, s);
}

// TCI_SKINNY_DMMA=0 keeps the CUDA-core streaming kernel (A/B measurements)
bool dmma_pass_disabled() {
  static const int off = [] {
    const char *e = getenv("TCI_SKINNY_DMMA");
    return e && e[0] == '0';
  }();
  return off;
}

// TCI_SKINNY_EXPAND=0 keeps the streaming kernel for expansion layouts (A/B)
bool expand_disabled() {
  static const int off = [] {
    const char *e = getenv("TCI_SKINNY_EXPAND");
    return e && e[0] == '0';
  }();
  return off;
}

}  // namespace

size_t skinny_smem_bytes(int K, int N, size_t esz) {
  return (size_t)(K * N + K * TB + TB * N) * esz;
}

cudaError_t launch_skinny(const SkinnyProblem &p0, cudaStream_t s, int64_t *launches) {
  SkinnyProblem p = p0;
  const bool cplx = p.dtype == TCI_C128;
  if (p.k_lo < 1 || p.K % p.k_lo) p.k_lo = 1;
  if (p.n_lo < 1 || p.N % p.n_lo) p.n_lo = 1;
  const size_t smem = skinny_smem_bytes(p.K, p.N, cplx ? 16 : 8);
  const int64_t blocks = p.nb[0] * p.nb[1] * ((p.nb[2] + TB - 1) / TB);
  if (blocks == 0) return cudaSuccess;
  if (expand_ok(p) && !expand_disabled()) {
    cudaError_t e = cplx ? launch_expand<true>(p, s) : launch_expand<false>(p, s);
    if (launches) ++*launches;
    return e;
  }
  // streaming variant: b2 unit-stride in the input, 16-byte aligned rows
  {
    const size_t es = cplx ? 16 : 8;
    bool ok = p.in_sb[2] == 1 && p.k_lo == 1 && ((uintptr_t)p.in % 16) == 0 && p.K <= kSkinnyMaxK &&
              p.N <= kSkinnyMaxN;
    const int64_t per = 16 / (int64_t)es;
    for (int k = 0; ok && k < p.K; k++) ok = p.in_koff[k] % per == 0;
    ok = ok && p.in_sb[0] % per == 0 && p.in_sb[1] % per == 0;
    const size_t ssm = (size_t)((cplx ? 3 : 1) * p.K * p.N + 1) * 8 + 2 * (size_t)p.K * TBS * es;
    if (ok && cplx && p.K <= 32 && p.N <= 32 && !dmma_pass_disabled()) {
      cudaError_t e = launch_dmma(p, s);   // FP64 tensor cores (DMMA), 3M
      if (launches) ++*launches;
      return e;
    }
    if (ok && ssm <= 200 * 1024) {
      cudaError_t e = cplx ? launch_stream<true>(p, s) : launch_stream<false>(p, s);
      if (launches) ++*launches;
      return e;
    }
  }
  if (blocks > 0x7fffffffLL || p.K > kSkinnyMaxK || p.N > kSkinnyMaxN || smem > 227 * 1024)
    return cudaErrorInvalidValue;
  cudaError_t e = cplx ? launch_c<true>(p, smem, blocks, s) : launch_c<false>(p, smem, blocks, s);
  if (launches) ++*launches;
  return e;
}

}  // namespace tci
