// permute.cu -- transpose kernel, Eq. (1) PAPER.md:167-174:
//   out[c_0..c_{n-1}] = in[c'] with c'[perm[k]] = c_k
// Pure data movement: bitwise exact. HBM-bound (roofline = measured copy
// bandwidth, 2 x bytes per element).
//
// The caller (plan.cpp) has fused adjacent legs that stay adjacent and
// dropped extent-1 legs, so the problem is `n` fused out legs with the input
// stride of each. Two kernels:
//  * copy_rows: the out-fastest leg is also in-contiguous -> each thread
//    moves 16-byte vectors along contiguous runs.
//  * transpose_tiles: the out-fastest leg j is strided in the input and some
//    other leg i is in-contiguous -> a (TI x TJ) tile is read along i with
//    16-byte loads into padded shared memory and written along j with
//    16-byte stores; every other leg indexes the tile grid.
#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

struct PermArgs {
  int nb;                        // batch legs (excluding i, j)
  int64_t bshape[kMaxOrder];
  int64_t b_in[kMaxOrder], b_out[kMaxOrder];
  int64_t ni, nj;                // extents of the tile legs
  int64_t i_in, i_out;           // strides: i is in-contiguous (i_in == 1)
  int64_t j_in, j_out;           // j is out-contiguous (j_out == 1)
  int64_t tiles_i, tiles_j;
  const char *in;
  char *out;
};

template <int ESZ, int VEC, int T>
__global__ void __launch_bounds__(256) transpose_tiles(const PermArgs a) {
  // element type of one vector
  using V = typename std::conditional<
      ESZ * VEC == 16, int4,
      typename std::conditional<ESZ * VEC == 8, int2, int>::type>::type;
  using E = typename std::conditional<ESZ == 16, int4,
                                      typename std::conditional<ESZ == 8, int2, int>::type>::type;
  // tile stored [j][i]; a one-element pad makes the pitch an odd number of
  // elements, so the column reads of the store phase are bank-conflict free
  __shared__ E tile[T][T + 1];

  int64_t bid = blockIdx.x;
  const int64_t tj = bid % a.tiles_j; bid /= a.tiles_j;
  const int64_t ti = bid % a.tiles_i; bid /= a.tiles_i;
  int64_t in_off = 0, out_off = 0;
  for (int k = a.nb - 1; k >= 0; k--) {
    const int64_t c = bid % a.bshape[k];
    bid /= a.bshape[k];
    in_off += c * a.b_in[k];
    out_off += c * a.b_out[k];
  }
  const int64_t i0 = ti * T, j0 = tj * T;
  const E *in = reinterpret_cast<const E *>(a.in) + in_off;
  E *out = reinterpret_cast<E *>(a.out) + out_off;
  constexpr int CPR = T / VEC;            // vectors per tile row
  constexpr int ROWS = 256 / CPR;         // rows per pass
  const int tid = threadIdx.x;
  // load phase: rows j, 16-byte vectors along the in-contiguous leg i
#pragma unroll
  for (int r = tid / CPR; r < T; r += ROWS) {
    const int iv = (tid % CPR) * VEC;
    const int64_t gi = i0 + iv, gj = j0 + r;
    if (gj < a.nj && gi < a.ni) {
      const E *src = in + gj * a.j_in + gi;
      if (VEC > 1 && gi + VEC <= a.ni) {
        V v = __ldg(reinterpret_cast<const V *>(src));
        const E *ve = reinterpret_cast<const E *>(&v);
#pragma unroll
        for (int e = 0; e < VEC; e++) tile[r][iv + e] = ve[e];
      } else {
        for (int e = 0; e < VEC && gi + e < a.ni; e++) tile[r][iv + e] = src[e];
      }
    }
  }
  __syncthreads();
  // store phase: consecutive threads -> consecutive j (out-contiguous):
  // each warp writes 32 consecutive elements (128-512 contiguous bytes)
  constexpr int SROWS = 256 / T;
#pragma unroll
  for (int r = tid / T; r < T; r += SROWS) {
    const int jl = tid % T;
    const int64_t gi = i0 + r, gj = j0 + jl;
    if (gi < a.ni && gj < a.nj) out[gi * a.i_out + gj] = tile[jl][r];
  }
}

struct RowArgs {
  int nb;
  int64_t bshape[kMaxOrder];
  int64_t b_in[kMaxOrder];
  int64_t run;          // contiguous run length (elements), out rows are contiguous
  int64_t rows;
  int64_t vec_per_row;
  const char *in;
  char *out;
};

template <int ESZ, int VEC>
__global__ void __launch_bounds__(256) copy_rows(const RowArgs a) {
  using E = typename std::conditional<ESZ == 16, int4,
                                      typename std::conditional<ESZ == 8, int2, int>::type>::type;
  using V = typename std::conditional<
      ESZ * VEC == 16, int4,
      typename std::conditional<ESZ * VEC == 8, int2, int>::type>::type;
  const int64_t total = a.rows * a.vec_per_row;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = idx / a.vec_per_row;
    const int64_t v = idx % a.vec_per_row;
    const int64_t out_row = row;
    int64_t in_off = 0;
    for (int k = a.nb - 1; k >= 0; k--) {
      const int64_t c = row % a.bshape[k];
      row /= a.bshape[k];
      in_off += c * a.b_in[k];
    }
    const E *src = reinterpret_cast<const E *>(a.in) + in_off + v * VEC;
    E *dst = reinterpret_cast<E *>(a.out) + out_row * a.run + v * VEC;
    if (VEC > 1 && (v + 1) * VEC <= a.run) {
      *reinterpret_cast<V *>(dst) = *reinterpret_cast<const V *>(src);
    } else {
      for (int e = 0; e < VEC && v * VEC + e < a.run; e++) dst[e] = src[e];
    }
  }
}

template <int ESZ>
cudaError_t launch_typed(const PermuteProblem &p, cudaStream_t s, int64_t *launches) {
  const int n = p.n;
  int64_t out_stride[kMaxOrder];
  {
    int64_t st = 1;
    for (int k = n - 1; k >= 0; k--) { out_stride[k] = st; st *= p.shape_out[k]; }
  }
  constexpr int VMAX = 16 / ESZ;
  auto aligned = [&](const void *ptr) { return ((uintptr_t)ptr % 16) == 0; };
  if (n == 0 || p.in_stride_for_out[n - 1] == 1) {
    RowArgs a{};
    a.run = n ? p.shape_out[n - 1] : 1;
    a.nb = n ? n - 1 : 0;
    a.rows = 1;
    bool vec_ok = aligned(p.in) && aligned(p.out) && (a.run % VMAX == 0);
    for (int k = 0; k < a.nb; k++) {
      a.bshape[k] = p.shape_out[k];
      a.b_in[k] = p.in_stride_for_out[k];
      a.rows *= p.shape_out[k];
      if (a.b_in[k] % VMAX) vec_ok = false;
    }
    a.in = static_cast<const char *>(p.in);
    a.out = static_cast<char *>(p.out);
    const int vec = vec_ok ? VMAX : 1;
    a.vec_per_row = (a.run + vec - 1) / vec;
    const int64_t total = a.rows * a.vec_per_row;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
    if (vec_ok) copy_rows<ESZ, VMAX><<<(unsigned)blocks, 256, 0, s>>>(a);
    else copy_rows<ESZ, 1><<<(unsigned)blocks, 256, 0, s>>>(a);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  // tile transpose between j = out-fastest leg and i = the in-contiguous leg
  int li = -1;
  for (int k = 0; k < n - 1; k++)
    if (p.in_stride_for_out[k] == 1) li = k;
  const int lj = n - 1;
  if (li < 0) {
    // no unit-stride input leg (cannot happen for a fused dense input): use rows
    return cudaErrorInvalidValue;
  }
  PermArgs a{};
  a.ni = p.shape_out[li];
  a.nj = p.shape_out[lj];
  a.i_in = 1;
  a.i_out = out_stride[li];
  a.j_in = p.in_stride_for_out[lj];
  a.j_out = 1;
  a.nb = 0;
  bool vec_ok = aligned(p.in) && (a.ni % VMAX == 0) && (a.j_in % VMAX == 0);
  int64_t nbt = 1;
  for (int k = 0; k < n; k++) {
    if (k == li || k == lj) continue;
    a.bshape[a.nb] = p.shape_out[k];
    a.b_in[a.nb] = p.in_stride_for_out[k];
    a.b_out[a.nb] = out_stride[k];
    if (a.b_in[a.nb] % VMAX) vec_ok = false;
    nbt *= p.shape_out[k];
    a.nb++;
  }
  constexpr int T = (ESZ == 16) ? 32 : 64;
  a.tiles_i = (a.ni + T - 1) / T;
  a.tiles_j = (a.nj + T - 1) / T;
  a.in = static_cast<const char *>(p.in);
  a.out = static_cast<char *>(p.out);
  const int64_t blocks = nbt * a.tiles_i * a.tiles_j;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  if (vec_ok) transpose_tiles<ESZ, VMAX, T><<<(unsigned)blocks, 256, 0, s>>>(a);
  else transpose_tiles<ESZ, 1, T><<<(unsigned)blocks, 256, 0, s>>>(a);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_permute(const PermuteProblem &p, cudaStream_t s, int64_t *launches) {
  if (p.total == 0) return cudaSuccess;
  switch (p.esize) {
    case 4: return launch_typed<4>(p, s, launches);
    case 8: return launch_typed<8>(p, s, launches);
    case 16: return launch_typed<16>(p, s, launches);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_copy(void *dst, const void *src, size_t bytes, cudaStream_t s, int64_t *launches) {
  (void)launches;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s);
}

}  // namespace tci
