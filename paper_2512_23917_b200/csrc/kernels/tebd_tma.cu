// tebd_tma.cu -- TEBD theta = (A.B).U for d = 2, float64 (SURVEY 8(a8),
// BASELINE config 3 "with TMA-fused permutes", reading
// R16) with every operand tile fetched by TMA multi-dimensional boxes
// straight out of the natural (A[a,s,b], B[b,t,c]) or physical-first
// (A[s,a,b], B[t,b,c]) layouts: the matricizing permute is the copy engine's
// address generation, no transposed copy exists anywhere.
//
//  * CTA tile: 64 a x 2 s rows by 2 t x 64 c columns (the four (s,t) gate
//    inputs of 64 x 64 (a,c) pairs), K = b in steps of 16, 4-stage mbarrier
//    ring filled by one thread: A as ONE 3-D box (16 b, 2 s, 64 a) -- or
//    (16 b, 64 a, 2 s) physical-first -- and B as eight 3-D boxes
//    (16 c, 1 t, 16 b) / (16 c, 16 b, 1 t), all SWIZZLE_128B (1 KB atoms of
//    8 rows x 128 B). Out-of-range a / b / c (ragged chi) arrive as zeros.
//  * FP64 DMMA m8n8k4, 8 warps of 64 x 32, k consumed in the same order as
//    the plain GEMM kernel (groups of 4 ascending), so an identity gate
//    gives A.B bitwise. (Permuting each DMMA's k values to {0,1,4,5}, ...
//    would spread a B fragment's four rows over both 64-byte halves of the
//    swizzled row space -- two wavefronts instead of four -- at the price of
//    that bitwise equality; shared memory is not the bound here: 256
//    wavefronts against 1024 DMMA cycles per k-step and CTA.)
//  * epilogue: the C tile is staged in shared memory and each thread applies
//    the 4 x 4 gate to (a, c) pairs (theta[a,p,q,c] at the caller's strides).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace {

constexpr int kBM = 128, kBN = 128, kBK = 16, kST = 4, kNT = 256;
constexpr int kABytes = kBM * kBK * 8;   // 16 KB: 128 rows x 128 B
constexpr int kBBytes = kBK * kBN * 8;   // 16 KB: 8 sub-tiles of 16 k x 16 c
constexpr int kStage = kABytes + kBBytes;
constexpr int kPC = kBN + 1;             // staged C pitch (doubles)
constexpr int kSmem = 1024 + std::max(kST * kStage + 8 * kST, kBM * kPC * 8);

struct TebdTmaArgs {
  int64_t chi_a, chi_b, chi_c;
  int pfA;                  // A rows are (s, a) instead of (a, s)
  int pfB;                  // B's map lists (c, b, t) instead of (c, t, b)
  int tiles_m, tiles_n;
  const double *U;
  int64_t u[4];             // strides of U[p, q, s, t]
  double *T;
  int64_t t[4];             // strides of theta over (a, p, q, c)
};

__device__ __forceinline__ void tma3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// byte offset of A(row r, k) in a stage (128-byte rows, 16-byte chunks XOR row % 8)
__device__ __forceinline__ uint32_t a_off(int r, int k) {
  return (uint32_t)(r * 128 + ((((k >> 1) ^ r) & 7) << 4) + ((k & 1) << 3));
}
// byte offset of B(k, n = t * 64 + c): sub-tile (t, c / 16) of 16 rows k x 16 doubles
__device__ __forceinline__ uint32_t b_off(int k, int n) {
  const int st = ((n >> 6) << 2) + ((n & 63) >> 4), cw = n & 15;
  return (uint32_t)(kABytes + st * 2048 + k * 128 + ((((cw >> 1) ^ k) & 7) << 4) + ((cw & 1) << 3));
}
// the k index lane-column lc uses in DMMA k-step kk of a 16-wide stage
__device__ __forceinline__ int kperm(int kk, int lc) { return 4 * kk + lc; }

__global__ void __launch_bounds__(kNT, 1) tebd_tma_kernel(const __grid_constant__ CUtensorMap mA,
                                                        const __grid_constant__ CUtensorMap mB,
                                                        const __grid_constant__ TebdTmaArgs p) {
  extern __shared__ uint8_t raw[];
  const uint32_t base_u = smem_u32(raw);
  uint8_t *sm = raw + (((base_u + 1023u) & ~1023u) - base_u);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + kST * kStage);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile_m = blockIdx.x / p.tiles_n, tile_n = blockIdx.x % p.tiles_n;
  const int a0 = tile_m * 64, c0 = tile_n * 64;
  const int KT = (int)((p.chi_b + kBK - 1) / kBK);

  if (tid == 0) {
    for (int s = 0; s < kST; s++) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int kt, int s) {   // thread 0
    uint8_t *st = sm + s * kStage;
    const int b0 = kt * kBK;
    mbar_expect_tx(&full[s], kStage);
    if (p.pfA)
      tma3d(st, &mA, &full[s], b0, a0, 0);
    else
      tma3d(st, &mA, &full[s], b0, 0, a0);
    // B boxes of 16 c x 16 b for one t: coordinates (c, t, b) natural,
    // (c, b, t) physical-first (the map lists the dims slowest-last)
#pragma unroll
    for (int t = 0; t < 2; t++)
#pragma unroll
      for (int cc = 0; cc < 4; cc++) {
        uint8_t *dst = st + kABytes + (t * 4 + cc) * 2048;
        if (p.pfB)
          tma3d(dst, &mB, &full[s], c0 + 16 * cc, b0, t);
        else
          tma3d(dst, &mB, &full[s], c0 + 16 * cc, t, b0);
      }
  };
  if (tid == 0)
    for (int s = 0; s < kST && s < KT; s++) issue(s, s);

  const int wm0 = (warp >> 2) * 64, wn0 = (warp & 3) * 32;
  const int lr = lane >> 2, lc = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; kt++) {
    const int s = kt % kST;
    mbar_wait(&full[s], (uint32_t)((kt / kST) & 1));
    const uint8_t *st = sm + s * kStage;
#pragma unroll
    for (int kk = 0; kk < kBK / 4; kk++) {
      const int k = kperm(kk, lc);
      double fa[8], fb[4];
#pragma unroll
      for (int i = 0; i < 8; i++) fa[i] = *reinterpret_cast<const double *>(st + a_off(wm0 + i * 8 + lr, k));
#pragma unroll
      for (int j = 0; j < 4; j++) fb[j] = *reinterpret_cast<const double *>(st + b_off(k, wn0 + j * 8 + lr));
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) dmma884(acc[i][j], fa[i], fb[j]);
    }
    __syncthreads();   // every warp is done with stage s
    if (tid == 0 && kt + kST < KT) {
      fence_proxy_async_smem();   // generic reads of the stage before the async-proxy refill
      issue(kt + kST, s);
    }
  }

  // ---- epilogue: C tile through shared memory, then the gate per (a, c) ----
  __syncthreads();
  double *Cs = reinterpret_cast<double *>(sm);
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int m = wm0 + i * 8 + lr, n = wn0 + j * 8 + 2 * lc;
      Cs[m * kPC + n] = acc[i][j][0];
      Cs[m * kPC + n + 1] = acc[i][j][1];
    }
  double u[2][2][2][2];
#pragma unroll
  for (int pp = 0; pp < 2; pp++)
#pragma unroll
    for (int q = 0; q < 2; q++)
#pragma unroll
      for (int s_ = 0; s_ < 2; s_++)
#pragma unroll
        for (int t_ = 0; t_ < 2; t_++) u[pp][q][s_][t_] = p.U[pp * p.u[0] + q * p.u[1] + s_ * p.u[2] + t_ * p.u[3]];
  __syncthreads();
  for (int idx = tid; idx < 64 * 64; idx += kNT) {
    const int al = idx >> 6, cl = idx & 63;
    const int64_t a = a0 + al, c = c0 + cl;
    if (a >= p.chi_a || c >= p.chi_c) continue;
    double x[2][2];
#pragma unroll
    for (int s_ = 0; s_ < 2; s_++) {
      const int r = p.pfA ? s_ * 64 + al : 2 * al + s_;
#pragma unroll
      for (int t_ = 0; t_ < 2; t_++) x[s_][t_] = Cs[r * kPC + t_ * 64 + cl];
    }
    double *T = p.T + a * p.t[0] + c * p.t[3];
#pragma unroll
    for (int pp = 0; pp < 2; pp++)
#pragma unroll
      for (int q = 0; q < 2; q++) {
        double th = 0.0;
#pragma unroll
        for (int s_ = 0; s_ < 2; s_++)
#pragma unroll
          for (int t_ = 0; t_ < 2; t_++) th = fma(u[pp][q][s_][t_], x[s_][t_], th);
        T[pp * p.t[1] + q * p.t[2]] = th;
      }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tebd_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 3-D float64 map over base with dims d (innermost first, d[0] unit stride),
// byte strides of dims 1 and 2, box b, SWIZZLE_128B (b[0] = 16 doubles)
bool map3(CUtensorMap *m, const double *base, const uint64_t (&d)[3], const uint64_t (&st)[2],
          const uint32_t (&b)[3]) {
  auto enc = tebd_encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {d[0], d[1], d[2]};
  const cuuint64_t strides[2] = {st[0], st[1]};
  const cuuint32_t box[3] = {b[0], b[1], b[2]};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// TMA requirements on top of tebd_fused_supported (unit-stride b in A and c
// in B, 16-byte aligned bases, even strides): byte strides multiples of 16
bool tebd_tma_supported(const TebdProblem &t) {
  auto m16 = [](int64_t elems) { return (elems * 8) % 16 == 0; };
  return t.d == 2 && t.a_b == 1 && t.b_c == 1 && ((uintptr_t)t.A % 16) == 0 && ((uintptr_t)t.B % 16) == 0 &&
         m16(t.a_a) && m16(t.a_s) && m16(t.b_b) && m16(t.b_t) && t.chi_a >= 1 && t.chi_b >= 1 && t.chi_c >= 1 &&
         t.chi_a <= (1ll << 31) && t.chi_b <= (1ll << 31) && t.chi_c <= (1ll << 31);
}

cudaError_t launch_tebd_tma(const TebdProblem &t, cudaStream_t s, int64_t *launches) {
  CUtensorMap mA, mB;
  const bool pfA = t.a_s > t.a_a, pfB = t.b_t > t.b_b;
  bool ok;
  if (pfA)   // A[s][a][b]: dims (b, a, s)
    ok = map3(&mA, t.A, {(uint64_t)t.chi_b, (uint64_t)t.chi_a, 2}, {(uint64_t)t.a_a * 8, (uint64_t)t.a_s * 8},
              {16, 64, 2});
  else       // A[a][s][b]: dims (b, s, a)
    ok = map3(&mA, t.A, {(uint64_t)t.chi_b, 2, (uint64_t)t.chi_a}, {(uint64_t)t.a_s * 8, (uint64_t)t.a_a * 8},
              {16, 2, 64});
  if (ok) {
    if (pfB)   // B[t][b][c]: dims (c, b, t)
      ok = map3(&mB, t.B, {(uint64_t)t.chi_c, (uint64_t)t.chi_b, 2}, {(uint64_t)t.b_b * 8, (uint64_t)t.b_t * 8},
                {16, 16, 1});
    else       // B[b][t][c]: dims (c, t, b)
      ok = map3(&mB, t.B, {(uint64_t)t.chi_c, 2, (uint64_t)t.chi_b}, {(uint64_t)t.b_t * 8, (uint64_t)t.b_b * 8},
                {16, 1, 16});
  }
  if (!ok) return cudaErrorNotSupported;
  TebdTmaArgs a{};
  a.chi_a = t.chi_a;
  a.chi_b = t.chi_b;
  a.chi_c = t.chi_c;
  a.pfA = pfA ? 1 : 0;
  a.pfB = pfB ? 1 : 0;
  a.tiles_m = (int)((t.chi_a + 63) / 64);
  a.tiles_n = (int)((t.chi_c + 63) / 64);
  a.U = t.U;
  a.u[0] = t.u_p; a.u[1] = t.u_q; a.u[2] = t.u_s; a.u[3] = t.u_t;
  a.T = t.T;
  a.t[0] = t.t_a; a.t[1] = t.t_p; a.t[2] = t.t_q; a.t[3] = t.t_c;
  cudaError_t e = ensure_smem_attr((const void *)tebd_tma_kernel, kSmem);
  if (e != cudaSuccess) return e;
  tebd_tma_kernel<<<(unsigned)((int64_t)a.tiles_m * a.tiles_n), kNT, kSmem, s>>>(mA, mB, a);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tci
