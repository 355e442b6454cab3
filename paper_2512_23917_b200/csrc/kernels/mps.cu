// mps.cu -- MPS overlap / norm transfer chain in ONE kernel (SURVEY 8(a9),
// config 1; chain definition DESIGN.md R17):
//   E_0 = [[1]];  X[z,s,y] = sum_x E[x,z] bra_i[x,s,y];  E'[y,w] = sum_{z,s} X[z,s,y] ket_i[z,s,w]
// for i = 0..n-1, result E_n (shape [chi_bra_n, chi_ket_n]).
// At chi = 16, d = 2 the whole chain is 46,808 MACs: launch latency, not
// FLOPs or bytes, is the bound, so the chain runs in a single CTA with E and
// X resident in shared memory; each step is one block-wide pass over the
// output elements (every element summed in ascending index order, as the
// oracle's contract does), separated by __syncthreads. Bilinear: no complex
// conjugation (R9); conjugate the bra beforehand for the Hermitian overlap.
#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

template <bool CPLX>
struct MT;
template <>
struct MT<false> {
  using T = double;
  static __device__ __forceinline__ T zero() { return 0.0; }
  static __device__ __forceinline__ T one() { return 1.0; }
  static __device__ __forceinline__ T mac(T c, T a, T b) { return fma(a, b, c); }
};
template <>
struct MT<true> {
  using T = double2;
  static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ T one() { return make_double2(1.0, 0.0); }
  static __device__ __forceinline__ T mac(T c, T a, T b) {
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(-a.y, b.y, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.y = fma(a.y, b.x, c.y);
    return c;
  }
};

template <bool CPLX>
__global__ void __launch_bounds__(256) mps_overlap_kernel(const __grid_constant__ MpsChain ch) {
  using O = MT<CPLX>;
  using T = typename O::T;
  extern __shared__ __align__(16) char sm[];
  T *E = reinterpret_cast<T *>(sm);                 // [kMpsMaxChi * kMpsMaxChi]
  T *X = E + kMpsMaxChi * kMpsMaxChi;               // [kMpsMaxChi * kMpsMaxD * kMpsMaxChi]
  T *S = X + kMpsMaxChi * kMpsMaxD * kMpsMaxChi;   // all site tensors (when they fit)
  const int tid = threadIdx.x;
  // stage every site tensor in shared memory up front: the chain is a
  // serial dependency, so global-load latency per step would dominate
  const bool staged = ch.staged_elems > 0;
  if (staged) {
    int off = 0, lb = 1, lk = 1;
    for (int i = 0; i < ch.n; i++) {
      const int nbi = lb * ch.d[i] * ch.bra_r[i], nki = lk * ch.d[i] * ch.ket_r[i];
      const T *Bg = reinterpret_cast<const T *>(ch.bra[i]);
      const T *Kg = reinterpret_cast<const T *>(ch.ket[i]);
      for (int e = tid; e < nbi; e += blockDim.x) S[off + e] = Bg[e];
      for (int e = tid; e < nki; e += blockDim.x) S[off + nbi + e] = Kg[e];
      off += nbi + nki;
      lb = ch.bra_r[i];
      lk = ch.ket_r[i];
    }
  }
  if (tid == 0) E[0] = O::one();
  int cb = 1, ck = 1;                               // current bra / ket bonds (E is cb x ck)
  int soff = 0;
  __syncthreads();
  for (int i = 0; i < ch.n; i++) {
    const int d = ch.d[i], nb = ch.bra_r[i], nk = ch.ket_r[i];
    const T *Bi = staged ? S + soff : reinterpret_cast<const T *>(ch.bra[i]);
    const T *Ki = staged ? S + soff + cb * d * nb : reinterpret_cast<const T *>(ch.ket[i]);
    soff += cb * d * nb + ck * d * nk;
    // X[z,s,y] = sum_x E[x,z] bra[x,s,y]   (bra is [cb, d, nb])
    for (int o = tid; o < ck * d * nb; o += blockDim.x) {
      const int z = o / (d * nb), s = (o / nb) % d, y = o % nb;
      T acc = O::zero();
      for (int x = 0; x < cb; x++) acc = O::mac(acc, E[x * ck + z], Bi[(x * d + s) * nb + y]);
      X[o] = acc;
    }
    __syncthreads();
    // E'[y,w] = sum_{z,s} X[z,s,y] ket[z,s,w]   (ket is [ck, d, nk])
    for (int o = tid; o < nb * nk; o += blockDim.x) {
      const int y = o / nk, w = o % nk;
      T acc = O::zero();
      for (int z = 0; z < ck; z++)
        for (int s = 0; s < d; s++) acc = O::mac(acc, X[(z * d + s) * nb + y], Ki[(z * d + s) * nk + w]);
      E[o] = acc;
    }
    __syncthreads();
    cb = nb;
    ck = nk;
  }
  T *out = reinterpret_cast<T *>(ch.out);
  for (int o = tid; o < cb * ck; o += blockDim.x) out[o] = E[o];
}

}  // namespace

cudaError_t launch_mps_overlap(const MpsChain &ch, cudaStream_t s, int64_t *launches) {
  const bool cplx = ch.dtype == TCI_C128;
  const size_t es = cplx ? 16 : 8;
  const size_t smem = (size_t)(kMpsMaxChi * kMpsMaxChi + kMpsMaxChi * kMpsMaxD * kMpsMaxChi + ch.staged_elems) * es;
  cudaError_t e;
  if (cplx) {
    e = cudaFuncSetAttribute(mps_overlap_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    mps_overlap_kernel<true><<<1, 256, smem, s>>>(ch);
  } else {
    e = cudaFuncSetAttribute(mps_overlap_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    mps_overlap_kernel<false><<<1, 256, smem, s>>>(ch);
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tci
