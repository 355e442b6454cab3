// gemm_thin.cu -- the HBM-bound corners of the GEMM over fused legs (SURVEY
// 8(a4)): products where one of M, N, K is tiny. A tensor-core tile
// (128x128x16) would compute mostly padding there, while the work is bound
// by streaming the one large operand (or the output) once:
//   * thin  (min(M, N) <= 32 real / 16 complex): C[m, n] = sum_k A[m, k] B[k, n], N thin
//     after an operand swap (C^T = B^T A^T); B's K-chunk is staged in shared
//     memory and every row of A is read once, coalesced along whichever of m
//     or k is contiguous (thread per row, or warp per row with a fixed-order
//     shuffle reduction). Split-K partials (fp64) use the planner's chunks.
//   * outer (K <= 16): thread per output column, rows of a 16-row tile from
//     shared memory; each output element is written once, coalesced.
// Products are accumulated in fp64 for every dtype (fp32 inputs are widened
// exactly, R20), in ascending k order: deterministic.
#include <algorithm>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

template <typename E>
struct TOps;
template <>
struct TOps<float> {
  using Acc = double;
  static __device__ __forceinline__ Acc zero() { return 0.0; }
  static __device__ __forceinline__ Acc wide(float a) { return (double)a; }
  static __device__ __forceinline__ void mac(Acc &c, Acc a, Acc b) { c = fma(a, b, c); }
  static __device__ __forceinline__ float out(Acc c) { return (float)c; }
  static __device__ __forceinline__ Acc shfl(Acc v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
  static __device__ __forceinline__ void add(Acc &c, Acc v) { c += v; }
};
template <>
struct TOps<double> {
  using Acc = double;
  static __device__ __forceinline__ Acc zero() { return 0.0; }
  static __device__ __forceinline__ Acc wide(double a) { return a; }
  static __device__ __forceinline__ void mac(Acc &c, Acc a, Acc b) { c = fma(a, b, c); }
  static __device__ __forceinline__ double out(Acc c) { return c; }
  static __device__ __forceinline__ Acc shfl(Acc v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
  static __device__ __forceinline__ void add(Acc &c, Acc v) { c += v; }
};
struct CplxOps {
  using Acc = double2;
  static __device__ __forceinline__ Acc zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ void mac(Acc &c, Acc a, Acc b) {
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(-a.y, b.y, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.y = fma(a.y, b.x, c.y);
  }
  static __device__ __forceinline__ Acc shfl(Acc v, int o) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o));
  }
  static __device__ __forceinline__ void add(Acc &c, Acc v) {
    c.x += v.x;
    c.y += v.y;
  }
};
template <>
struct TOps<float2> : CplxOps {
  static __device__ __forceinline__ Acc wide(float2 a) { return make_double2(a.x, a.y); }
  static __device__ __forceinline__ float2 out(Acc c) { return make_float2((float)c.x, (float)c.y); }
};
template <>
struct TOps<double2> : CplxOps {
  static __device__ __forceinline__ Acc wide(double2 a) { return a; }
  static __device__ __forceinline__ double2 out(Acc c) { return c; }
};

struct ThinArgs {
  int64_t M, N, K;                 // N <= 32 (16 complex; thin) or K <= 16 (outer)
  const void *A; int64_t a_sm, a_sk;
  const void *B; int64_t b_sk, b_sn;
  void *C; int64_t c_sm, c_sn;
  const int64_t *c_row, *c_col;    // gamma-order scatter tables (or nullptr)
  void *P; int64_t p_sm, p_sn, p_sz;   // split-K partials (fp64), or P == nullptr
  int64_t k_chunk;
};

constexpr int TT = 256;      // threads
constexpr int KC = 128;      // K rows of B staged per step (thin)

// thin, A m-contiguous (a_sm == 1): thread per row m
template <typename E, int NN>
__global__ void __launch_bounds__(TT) thin_mfast(const ThinArgs a) {
  using O = TOps<E>;
  using Acc = typename O::Acc;
  __shared__ Acc Bs[KC][NN];
  const int64_t m = blockIdx.x * (int64_t)TT + threadIdx.x;
  const int64_t kb = (int64_t)blockIdx.z * a.k_chunk;
  const int64_t ke = min(a.K, kb + a.k_chunk);
  const E *A = static_cast<const E *>(a.A);
  const E *B = static_cast<const E *>(a.B);
  Acc acc[NN];
#pragma unroll
  for (int n = 0; n < NN; n++) acc[n] = O::zero();
  for (int64_t k0 = kb; k0 < ke; k0 += KC) {
    const int kc = (int)min((int64_t)KC, ke - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < KC * NN; i += TT) {
      int k, n;
      if (a.b_sn == 1) { k = i / NN; n = i % NN; } else { n = i / KC; k = i % KC; }
      Bs[k][n] = (k < kc && n < a.N) ? O::wide(B[(k0 + k) * a.b_sk + n * a.b_sn]) : O::zero();
    }
    __syncthreads();
    if (m < a.M) {
      const E *Ap = A + m + k0 * a.a_sk;
#pragma unroll 4
      for (int k = 0; k < kc; k++) {
        const Acc x = O::wide(Ap[k * a.a_sk]);
#pragma unroll
        for (int n = 0; n < NN; n++) O::mac(acc[n], x, Bs[k][n]);
      }
    }
  }
  if (m >= a.M) return;
#pragma unroll
  for (int n = 0; n < NN; n++) {
    if (n >= a.N) break;
    if (a.P) static_cast<Acc *>(a.P)[blockIdx.z * a.p_sz + m * a.p_sm + n * a.p_sn] = acc[n];
    else static_cast<E *>(a.C)[a.c_row ? a.c_row[m] + a.c_col[n] : m * a.c_sm + n * a.c_sn] = O::out(acc[n]);
  }
}

// thin, A k-contiguous (a_sk == 1): warp per row m, lanes along k
template <typename E, int NN>
__global__ void __launch_bounds__(TT) thin_kfast(const ThinArgs a) {
  using O = TOps<E>;
  using Acc = typename O::Acc;
  __shared__ Acc Bs[NN][KC + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = blockIdx.x * (int64_t)(TT / 32) + warp;
  const int64_t kb = (int64_t)blockIdx.z * a.k_chunk;
  const int64_t ke = min(a.K, kb + a.k_chunk);
  const E *A = static_cast<const E *>(a.A);
  const E *B = static_cast<const E *>(a.B);
  Acc acc[NN];
#pragma unroll
  for (int n = 0; n < NN; n++) acc[n] = O::zero();
  for (int64_t k0 = kb; k0 < ke; k0 += KC) {
    const int kc = (int)min((int64_t)KC, ke - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < KC * NN; i += TT) {
      int k, n;
      if (a.b_sn == 1) { k = i / NN; n = i % NN; } else { n = i / KC; k = i % KC; }
      Bs[n][k] = (k < kc && n < a.N) ? O::wide(B[(k0 + k) * a.b_sk + n * a.b_sn]) : O::zero();
    }
    __syncthreads();
    if (m < a.M) {
      const E *Ap = A + m * a.a_sm + k0;
#pragma unroll 2
      for (int k = lane; k < kc; k += 32) {
        const Acc x = O::wide(Ap[k]);
#pragma unroll
        for (int n = 0; n < NN; n++) O::mac(acc[n], x, Bs[n][k]);
      }
    }
  }
  // fixed xor-tree reduction over the lanes
#pragma unroll
  for (int n = 0; n < NN; n++)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) O::add(acc[n], O::shfl(acc[n], o));
  if (m >= a.M || lane != 0) return;
#pragma unroll
  for (int n = 0; n < NN; n++) {
    if (n >= a.N) break;
    if (a.P) static_cast<Acc *>(a.P)[blockIdx.z * a.p_sz + m * a.p_sm + n * a.p_sn] = acc[n];
    else static_cast<E *>(a.C)[a.c_row ? a.c_row[m] + a.c_col[n] : m * a.c_sm + n * a.c_sn] = O::out(acc[n]);
  }
}

// outer: K <= 16; CTA = RM rows x 256 columns, thread per column with its
// K values of B in registers, A's RM x K tile in shared memory
constexpr int RM = 32;
template <typename E, int KK>
__global__ void __launch_bounds__(TT) outer_kernel(const ThinArgs a, int64_t tiles_n) {
  using O = TOps<E>;
  using Acc = typename O::Acc;
  __shared__ Acc As[RM][KK];
  const int64_t tn = blockIdx.x % tiles_n, tm = blockIdx.x / tiles_n;
  const int64_t m0 = tm * RM, n0 = tn * TT;
  const int K = (int)a.K;
  const E *A = static_cast<const E *>(a.A);
  const E *B = static_cast<const E *>(a.B);
  for (int i = threadIdx.x; i < RM * KK; i += TT) {
    const int r = i / KK, k = i % KK;
    As[r][k] = (m0 + r < a.M && k < K) ? O::wide(A[(m0 + r) * a.a_sm + k * a.a_sk]) : O::zero();
  }
  const int64_t n = n0 + threadIdx.x;
  Acc b[KK];
#pragma unroll
  for (int k = 0; k < KK; k++) b[k] = (k < K && n < a.N) ? O::wide(B[k * a.b_sk + n * a.b_sn]) : O::zero();
  __syncthreads();
  if (n >= a.N) return;
  E *C = static_cast<E *>(a.C);
  const int rows = (int)min((int64_t)RM, a.M - m0);
  for (int r = 0; r < rows; r++) {
    Acc acc = O::zero();
#pragma unroll
    for (int k = 0; k < KK; k++) O::mac(acc, As[r][k], b[k]);   // padded k: zeros
    C[a.c_row ? a.c_row[m0 + r] + a.c_col[n] : (m0 + r) * a.c_sm + n * a.c_sn] = O::out(acc);
  }
}

template <typename E, int NN>
cudaError_t launch_thin_nn(const ThinArgs &t, int splits, cudaStream_t s) {
  if (t.a_sm == 1 && t.a_sk != 1) {
    dim3 grid((unsigned)((t.M + TT - 1) / TT), 1, (unsigned)splits);
    thin_mfast<E, NN><<<grid, TT, 0, s>>>(t);
  } else {
    dim3 grid((unsigned)((t.M + TT / 32 - 1) / (TT / 32)), 1, (unsigned)splits);
    thin_kfast<E, NN><<<grid, TT, 0, s>>>(t);
  }
  return cudaGetLastError();
}

template <typename E>
cudaError_t launch_thin_t(const ThinArgs &t, int splits, cudaStream_t s) {
  if (t.N <= 1) return launch_thin_nn<E, 1>(t, splits, s);
  if (t.N <= 2) return launch_thin_nn<E, 2>(t, splits, s);
  if (t.N <= 4) return launch_thin_nn<E, 4>(t, splits, s);
  if (t.N <= 8) return launch_thin_nn<E, 8>(t, splits, s);
  if constexpr (sizeof(typename TOps<E>::Acc) == 16) {
    return launch_thin_nn<E, 16>(t, splits, s);   // complex: thin side <= 16
  } else {
    if (t.N <= 16) return launch_thin_nn<E, 16>(t, splits, s);
    return launch_thin_nn<E, 32>(t, splits, s);
  }
}

template <typename E>
cudaError_t launch_outer_t(const ThinArgs &t, cudaStream_t s) {
  const int64_t tn = (t.N + TT - 1) / TT, tm = (t.M + RM - 1) / RM;
  if (tn * tm > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const unsigned g = (unsigned)(tn * tm);
  if (t.K <= 1) outer_kernel<E, 1><<<g, TT, 0, s>>>(t, tn);
  else if (t.K <= 2) outer_kernel<E, 2><<<g, TT, 0, s>>>(t, tn);
  else if (t.K <= 4) outer_kernel<E, 4><<<g, TT, 0, s>>>(t, tn);
  else if (t.K <= 8) outer_kernel<E, 8><<<g, TT, 0, s>>>(t, tn);
  else outer_kernel<E, 16><<<g, TT, 0, s>>>(t, tn);
  return cudaGetLastError();
}

}  // namespace

bool gemm_thin_applies(const GemmProblem &p) {
  if (p.mode != 0 || p.M == 0 || p.N == 0) return false;
  // thin side up to 32 (complex: 16, register budget); real GEMM tiles waste >= 75 % there
  const int64_t thin_max = dtype_is_complex(p.dtype) ? 16 : 32;
  if (std::min(p.M, p.N) <= thin_max) return p.M < (1LL << 31) && p.N < (1LL << 31);
  return p.K <= 16 && p.splitk <= 1;
}

cudaError_t launch_gemm_thin(const GemmProblem &p, cudaStream_t s, int64_t *launches) {
  ThinArgs t{};
  const int splits = p.splitk > 1 ? p.splitk : 1;
  t.K = p.K;
  t.k_chunk = p.splitk > 1 ? p.k_chunk : p.K;
  const int64_t thin_max = dtype_is_complex(p.dtype) ? 16 : 32;   // as gemm_thin_applies
  const bool outer = std::min(p.M, p.N) > thin_max;
  // thin: make N the thin side (C^T = B^T A^T when M is the thin one)
  const bool swap = !outer && p.M < p.N;
  if (!swap) {
    t.M = p.M; t.N = p.N;
    t.A = p.A; t.a_sm = p.a_sm; t.a_sk = p.a_sk;
    t.B = p.B; t.b_sk = p.b_sk; t.b_sn = p.b_sn;
    t.c_sm = p.c_sm; t.c_sn = 1;
    t.c_row = p.c_row; t.c_col = p.c_col;
    t.p_sm = p.N; t.p_sn = 1;
  } else {
    t.M = p.N; t.N = p.M;
    t.A = p.B; t.a_sm = p.b_sn; t.a_sk = p.b_sk;
    t.B = p.A; t.b_sk = p.a_sk; t.b_sn = p.a_sm;
    t.c_sm = 1; t.c_sn = p.c_sm;
    t.c_row = p.c_col; t.c_col = p.c_row;
    t.p_sm = 1; t.p_sn = p.N;
  }
  // degenerate extents: a single row / column has no meaningful stride
  if (t.M == 1) t.a_sm = 0;
  if (t.K == 1) t.a_sk = 0;
  t.C = p.C;
  t.P = p.splitk > 1 ? p.partial : nullptr;
  t.p_sz = p.M * p.N;
  // loader choice needs one unit stride (a_sm == 1 -> thread per row)
  if (!(t.a_sm == 1 && t.a_sk != 1) && t.a_sk != 1 && t.K > 1 && !outer) {
    // neither stride is 1 after the swap: cannot happen for planner output
    return cudaErrorInvalidValue;
  }
  cudaError_t e;
  switch (p.dtype) {
    case TCI_R32: e = outer ? launch_outer_t<float>(t, s) : launch_thin_t<float>(t, splits, s); break;
    case TCI_R64: e = outer ? launch_outer_t<double>(t, s) : launch_thin_t<double>(t, splits, s); break;
    case TCI_C64: e = outer ? launch_outer_t<float2>(t, s) : launch_thin_t<float2>(t, splits, s); break;
    default: e = outer ? launch_outer_t<double2>(t, s) : launch_thin_t<double2>(t, splits, s); break;
  }
  if (launches) ++*launches;
  return e;
}

}  // namespace tci
