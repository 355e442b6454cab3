// vec.cu -- element-wise / reduction kernels for the Lanczos driver around
// H_eff and the TCI vector functions they realise:
//   norm (Frobenius, Eq. frob_norm), scale,
//   linear_combine, and the inner product <a|b> = sum conj?(a) b
//   (a full contraction to a scalar, with cplx_conj P:1235-1268).
// All HBM-bound. Reductions are deterministic: a fixed grid (4 x 148 CTAs),
// each CTA sums a fixed strided set of elements in a fixed order and writes
// one partial; a second single-CTA pass adds the partials in ascending order.
// Results are therefore bitwise reproducible run to run.
#include <algorithm>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

constexpr int RB = kReduceBlocks;   // reduction CTAs (4 per SM)
constexpr int RT = 256;

// block-wide sum in a fixed tree order
template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double (*sh)[RT]) {
#pragma unroll
  for (int i = 0; i < N; i++) sh[i][threadIdx.x] = v[i];
  __syncthreads();
  for (int s = RT / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
#pragma unroll
      for (int i = 0; i < N; i++) sh[i][threadIdx.x] += sh[i][threadIdx.x + s];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < N; i++) v[i] = sh[i][0];
}

// pass 1: per-CTA partials of sum |x|^2 (NV = 1) or sum conj?(a) b (NV = 2)
template <int MODE>   // 0: norm2 real/complex-as-reals, 1: inner complex, 2: inner real
__global__ void __launch_bounds__(RT) reduce_pass1(const double *a, const double *b, int64_t n_reals,
                                                   int conj_a, double *part) {
  __shared__ double sh[2][RT];
  double v[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * RT;
  if (MODE == 0) {
    for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n_reals; i += stride) v[0] = fma(a[i], a[i], v[0]);
  } else if (MODE == 2) {
    for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n_reals; i += stride) v[0] = fma(a[i], b[i], v[0]);
  } else {
    const double2 *a2 = reinterpret_cast<const double2 *>(a), *b2 = reinterpret_cast<const double2 *>(b);
    const double sg = conj_a ? -1.0 : 1.0;
#pragma unroll 4
    for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n_reals / 2; i += stride) {
      const double2 x = a2[i], y = b2[i];
      // (xr + i sg xi)(yr + i yi)
      v[0] = fma(x.x, y.x, v[0]);
      v[0] = fma(-sg * x.y, y.y, v[0]);
      v[1] = fma(x.x, y.y, v[1]);
      v[1] = fma(sg * x.y, y.x, v[1]);
    }
  }
  block_sum<2>(v, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = v[0];
    part[2 * blockIdx.x + 1] = v[1];
  }
}

__global__ void __launch_bounds__(RT) reduce_pass2(const double *part, int nb, double *out) {
  __shared__ double sh[2][RT];
  double v[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < nb; i += RT) {
    v[0] += part[2 * i];
    v[1] += part[2 * i + 1];
  }
  block_sum<2>(v, sh);
  if (threadIdx.x == 0) {
    out[0] = v[0];
    out[1] = v[1];
  }
}

// Several inner products <v_i|w> (i < m <= kMaxMI) in one pass: w is read
// once; each v_i's sum runs in exactly the order of reduce_pass1 / pass2 (same
// grid, same per-thread sequence, same trees), so every result is bitwise the
// single inner product's.
struct MiArgs {
  const double *v[kMaxMI];
  int m;
};

template <bool CPLX, int M>
__global__ void __launch_bounds__(RT) multi_inner_pass1(const __grid_constant__ MiArgs a, const double *w,
                                                        int64_t n_reals, int conj_a, double *part) {
  __shared__ double sh[2][RT];
  double acc[M][2];
#pragma unroll
  for (int i = 0; i < M; i++) acc[i][0] = acc[i][1] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * RT;
  if (CPLX) {
    const double2 *w2 = reinterpret_cast<const double2 *>(w);
    const double sg = conj_a ? -1.0 : 1.0;
#pragma unroll 2
    for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < n_reals / 2; e += stride) {
      const double2 y = w2[e];
      double2 x[M];
#pragma unroll
      for (int i = 0; i < M; i++) x[i] = reinterpret_cast<const double2 *>(a.v[i])[e];
#pragma unroll
      for (int i = 0; i < M; i++) {
        acc[i][0] = fma(x[i].x, y.x, acc[i][0]);
        acc[i][0] = fma(-sg * x[i].y, y.y, acc[i][0]);
        acc[i][1] = fma(x[i].x, y.y, acc[i][1]);
        acc[i][1] = fma(sg * x[i].y, y.x, acc[i][1]);
      }
    }
  } else {
#pragma unroll 2
    for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < n_reals; e += stride) {
      const double y = w[e];
#pragma unroll
      for (int i = 0; i < M; i++) acc[i][0] = fma(a.v[i][e], y, acc[i][0]);
    }
  }
#pragma unroll 1
  for (int i = 0; i < M; i++) {
    double v[2] = {acc[i][0], acc[i][1]};
    block_sum<2>(v, sh);
    if (threadIdx.x == 0) {
      part[(size_t)i * 2 * gridDim.x + 2 * blockIdx.x] = v[0];
      part[(size_t)i * 2 * gridDim.x + 2 * blockIdx.x + 1] = v[1];
    }
    __syncthreads();
  }
}

template <bool CPLX>
void multi_inner_launch(int m, const MiArgs &a, const double *w, int64_t n_reals, int conj_a, double *part,
                        cudaStream_t s) {
  switch (m) {
    case 1: multi_inner_pass1<CPLX, 1><<<RB, RT, 0, s>>>(a, w, n_reals, conj_a, part); break;
    case 2: multi_inner_pass1<CPLX, 2><<<RB, RT, 0, s>>>(a, w, n_reals, conj_a, part); break;
    case 3: multi_inner_pass1<CPLX, 3><<<RB, RT, 0, s>>>(a, w, n_reals, conj_a, part); break;
    case 4: multi_inner_pass1<CPLX, 4><<<RB, RT, 0, s>>>(a, w, n_reals, conj_a, part); break;
    case 5: multi_inner_pass1<CPLX, 5><<<RB, RT, 0, s>>>(a, w, n_reals, conj_a, part); break;
    case 6: multi_inner_pass1<CPLX, 6><<<RB, RT, 0, s>>>(a, w, n_reals, conj_a, part); break;
    case 7: multi_inner_pass1<CPLX, 7><<<RB, RT, 0, s>>>(a, w, n_reals, conj_a, part); break;
    default: multi_inner_pass1<CPLX, 8><<<RB, RT, 0, s>>>(a, w, n_reals, conj_a, part); break;
  }
}

// out = sum_j c_j in_j over up to kMaxLC inputs (complex coefficients);
// CPLX: elements are (re, im) pairs
struct LcArgs {
  const double *in[kMaxLC];
  double cr[kMaxLC], ci[kMaxLC];
  int m;
  double *out;
  int64_t n;   // elements (complex elements when CPLX)
};

template <bool CPLX>
__global__ void __launch_bounds__(RT) lincomb_kernel(const __grid_constant__ LcArgs a) {
  const int64_t stride = (int64_t)gridDim.x * RT;
  for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < a.n; i += stride) {
    if (CPLX) {
      double re = 0.0, im = 0.0;
      for (int j = 0; j < a.m; j++) {
        const double2 x = reinterpret_cast<const double2 *>(a.in[j])[i];
        re = fma(a.cr[j], x.x, re);
        re = fma(-a.ci[j], x.y, re);
        im = fma(a.cr[j], x.y, im);
        im = fma(a.ci[j], x.x, im);
      }
      reinterpret_cast<double2 *>(a.out)[i] = make_double2(re, im);
    } else {
      double r = 0.0;
      for (int j = 0; j < a.m; j++) r = fma(a.cr[j], a.in[j][i], r);
      a.out[i] = r;
    }
  }
}

}  // namespace

// sum |x_i|^2 (n_reals doubles) or sum conj?(a) b into out[2] (device), using
// part[2 * RB] device scratch
cudaError_t launch_reduce(int mode, const double *a, const double *b, int64_t n_reals, int conj_a,
                          double *part, double *out, cudaStream_t s, int64_t *launches) {
  if (mode == 0) reduce_pass1<0><<<RB, RT, 0, s>>>(a, b, n_reals, conj_a, part);
  else if (mode == 1) reduce_pass1<1><<<RB, RT, 0, s>>>(a, b, n_reals, conj_a, part);
  else reduce_pass1<2><<<RB, RT, 0, s>>>(a, b, n_reals, conj_a, part);
  reduce_pass2<<<1, RT, 0, s>>>(part, RB, out);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// [multi-inner partials: kMaxMI x 2 RB][multi-inner results: 2 x kMaxMIOut][single partials 2 RB][single result 2]
size_t reduce_scratch_bytes() {
  return (2 * RB * kMaxMI + 2 * kMaxMIOut + 2 * RB + 2) * sizeof(double);
}

// <v_i|w> for i < m (any m <= kMaxMIOut) into out[2 i] (device, the
// results region of the scratch), chunks of kMaxMI vectors per pass over w
cudaError_t launch_multi_inner(bool cplx, const double *const *v, int m, const double *w, int64_t n_reals, int conj_a,
                               double *scratch, double *out, cudaStream_t s, int64_t *launches) {
  if (m > kMaxMIOut) return cudaErrorInvalidValue;
  for (int i0 = 0; i0 < m; i0 += kMaxMI) {
    MiArgs a{};
    a.m = std::min(kMaxMI, m - i0);
    for (int i = 0; i < a.m; i++) a.v[i] = v[i0 + i];
    if (cplx) multi_inner_launch<true>(a.m, a, w, n_reals, conj_a, scratch, s);
    else multi_inner_launch<false>(a.m, a, w, n_reals, conj_a, scratch, s);
    for (int i = 0; i < a.m; i++) reduce_pass2<<<1, RT, 0, s>>>(scratch + (size_t)i * 2 * RB, RB, out + 2 * (i0 + i));
    if (launches) *launches += 1 + a.m;
  }
  return cudaGetLastError();
}

cudaError_t launch_lincomb(bool cplx, const double *const *in, const double *cr, const double *ci, int m,
                           double *out, int64_t n, cudaStream_t s, int64_t *launches) {
  LcArgs a{};
  a.m = m;
  a.out = out;
  a.n = n;
  for (int j = 0; j < m; j++) {
    a.in[j] = in[j];
    a.cr[j] = cr[j];
    a.ci[j] = ci ? ci[j] : 0.0;
  }
  const int64_t blocks = std::min<int64_t>((n + RT - 1) / RT, 148 * 8);
  if (blocks <= 0) return cudaSuccess;
  if (cplx) lincomb_kernel<true><<<(unsigned)blocks, RT, 0, s>>>(a);
  else lincomb_kernel<false><<<(unsigned)blocks, RT, 0, s>>>(a);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// out[r, c] = s[r] * in[r, c] (real scale s, r64 / c128 rows of `cols`
// elements): the diagonal S of an SVD absorbed into V^H (zip-up carry)
template <bool C>
__global__ void __launch_bounds__(RT) row_scale_kernel(const double *in, const double *s, double *out, int64_t rows,
                                                       int64_t cols) {
  const int64_t w = C ? 2 : 1, n = rows * cols * w;
  for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT)
    out[i] = s[i / (cols * w)] * in[i];
}

cudaError_t launch_row_scale(bool cplx, const double *in, const double *s, double *out, int64_t rows, int64_t cols,
                             cudaStream_t st, int64_t *launches) {
  const int64_t n = rows * cols * (cplx ? 2 : 1);
  const int64_t blocks = std::min<int64_t>((n + RT - 1) / RT, 148 * 8);
  if (blocks <= 0) return cudaSuccess;
  if (cplx) row_scale_kernel<true><<<(unsigned)blocks, RT, 0, st>>>(in, s, out, rows, cols);
  else row_scale_kernel<false><<<(unsigned)blocks, RT, 0, st>>>(in, s, out, rows, cols);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// complex conjugation: out[i] = (re, -im); in == out allowed.
// 16-byte elements, grid-stride, one load and one store per element.
__global__ void __launch_bounds__(RT) conj_kernel(const double2 *in, double2 *out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT) {
    const double2 v = in[i];
    out[i] = make_double2(v.x, -v.y);
  }
}

cudaError_t launch_conj(const void *in, void *out, int64_t n, cudaStream_t s, int64_t *launches) {
  const int64_t blocks = std::min<int64_t>((n + RT - 1) / RT, 148 * 8);
  if (blocks <= 0) return cudaSuccess;
  conj_kernel<<<(unsigned)blocks, RT, 0, s>>>(static_cast<const double2 *>(in), static_cast<double2 *>(out), n);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tci
