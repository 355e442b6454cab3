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

template <bool CPLX, int NPT>
cudaError_t launch_npt(const SkinnyProblem &p, size_t smem, int64_t blocks, cudaStream_t s) {
  auto k = skinny_kernel<CPLX, NPT>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
  if (blocks > 0x7fffffffLL || p.K > kSkinnyMaxK || p.N > kSkinnyMaxN || smem > 227 * 1024)
    return cudaErrorInvalidValue;
  cudaError_t e = cplx ? launch_c<true>(p, smem, blocks, s) : launch_c<false>(p, smem, blocks, s);
  if (launches) ++*launches;
  return e;
}

}  // namespace tci
