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
//    (16 b, 64 a, 2 s) physical-first -- SWIZZLE_128B, and B as sixteen
//    unswizzled 3-D boxes (8 c, 1 t, 16 b) / (8 c, 16 b, 1 t) of 64-byte
//    rows. Out-of-range a / b / c (ragged chi) arrive as zeros.
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
constexpr int kSmem = 1024 + std::max(kST * kStage + 16 * kST, kBM * kPC * 8);

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
// byte offset of B(k, n = t * 64 + c): sub-tile (t, c / 8) of 16 rows k x 8
// doubles, unswizzled: a DMMA B fragment (4 rows k x 8 n) reads 4 x 64 B
// that fall alternately into the two halves of the bank space -- two
// wavefronts, the minimum for 256 B
__device__ __forceinline__ uint32_t b_off(int k, int n) {
  const int st = ((n >> 6) << 3) + ((n & 63) >> 3), cw = n & 7;
  return (uint32_t)(kABytes + st * 1024 + k * 64 + cw * 8);
}
// the k index lane-column lc uses in DMMA k-step kk of a 16-wide stage
__device__ __forceinline__ int kperm(int kk, int lc) { return 4 * kk + lc; }

__global__ void __launch_bounds__(kNT + 32, 1) tebd_tma_kernel(const __grid_constant__ CUtensorMap mA,
                                                        const __grid_constant__ CUtensorMap mB,
                                                        const __grid_constant__ TebdTmaArgs p) {
  extern __shared__ uint8_t raw[];
  const uint32_t base_u = smem_u32(raw);
  uint8_t *sm = raw + (((base_u + 1023u) & ~1023u) - base_u);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + kST * kStage);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // grouped raster (as the DMMA GEMM): 8 M-tiles walk the N-tiles together,
  // so the B panels they share stay in L2
  constexpr int GROUP = 8;
  const int bid = blockIdx.x, per_group = GROUP * p.tiles_n;
  const int first_m = (bid / per_group) * GROUP;
  const int gsize = min(p.tiles_m - first_m, GROUP);
  const int tile_m = first_m + (bid % per_group) % gsize;
  const int tile_n = (bid % per_group) / gsize;
  const int a0 = tile_m * 64, c0 = tile_n * 64;
  const int KT = (int)((p.chi_b + kBK - 1) / kBK);

  uint64_t *empty = full + kST;
  if (tid == 0) {
    for (int s = 0; s < kST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNT / 32);   // one arrival per compute warp
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (tid >= kNT) {
    // ===== producer warp: the 17 boxes of each stage, kST stages ahead of
    // the compute warps (full / empty mbarriers; no block-wide barrier in
    // the main loop) =====
    if (lane == 0) {
      for (int kt = 0; kt < KT; kt++) {
        const int s = kt % kST;
        if (kt >= kST) mbar_wait(&empty[s], (uint32_t)(((kt / kST) - 1) & 1));
        uint8_t *st = sm + s * kStage;
        const int b0 = kt * kBK;
        fence_proxy_async_smem();
        mbar_expect_tx(&full[s], kStage);
        if (p.pfA)
          tma3d(st, &mA, &full[s], b0, a0, 0);
        else
          tma3d(st, &mA, &full[s], b0, 0, a0);
        // B boxes of 8 c x 16 b for one t: coordinates (c, t, b) natural,
        // (c, b, t) physical-first (the map lists the dims slowest-last)
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int t = j >> 3, cc = j & 7;
          uint8_t *dst = st + kABytes + j * 1024;
          if (p.pfB)
            tma3d(dst, &mB, &full[s], c0 + 8 * cc, b0, t);
          else
            tma3d(dst, &mB, &full[s], c0 + 8 * cc, t, b0);
        }
      }
    }
  }

  const int wm0 = (warp >> 2) * 64, wn0 = (warp & 3) * 32;
  const int lr = lane >> 2, lc = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  // fragments double-buffered in registers: k-step kk + 1's shared-memory
  // loads are in flight while kk's 32 DMMAs issue
  auto load_frags = [&](const uint8_t *st, int kk, double (&fa)[8], double (&fb)[4]) {
    const int k = kperm(kk, lc);
#pragma unroll
    for (int i = 0; i < 8; i++) fa[i] = *reinterpret_cast<const double *>(st + a_off(wm0 + i * 8 + lr, k));
#pragma unroll
    for (int j = 0; j < 4; j++) fb[j] = *reinterpret_cast<const double *>(st + b_off(k, wn0 + j * 8 + lr));
  };
  if (tid < kNT) {
    for (int kt = 0; kt < KT; kt++) {
      const int s = kt % kST;
      mbar_wait(&full[s], (uint32_t)((kt / kST) & 1));
      const uint8_t *st = sm + s * kStage;
      double fa[2][8], fb[2][4];
      load_frags(st, 0, fa[0], fb[0]);
#pragma unroll
      for (int kk = 0; kk < kBK / 4; kk++) {
        if (kk + 1 < kBK / 4) load_frags(st, kk + 1, fa[(kk + 1) & 1], fb[(kk + 1) & 1]);
#pragma unroll
        for (int i = 0; i < 8; i++)
#pragma unroll
          for (int j = 0; j < 4; j++) dmma884(acc[i][j], fa[kk & 1][i], fb[kk & 1][j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done with stage s
    }
  }

  // ---- epilogue: C tile through shared memory, then the gate per (a, c) ----
  __syncthreads();   // every stage consumed (and no TMA write in flight: all were waited on)
  double *Cs = reinterpret_cast<double *>(sm);
  if (tid < kNT)
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
  for (int idx = tid; tid < kNT && idx < 64 * 64; idx += kNT) {
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
          const uint32_t (&b)[3], bool swz) {
  auto enc = tebd_encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {d[0], d[1], d[2]};
  const cuuint64_t strides[2] = {st[0], st[1]};
  const cuuint32_t box[3] = {b[0], b[1], b[2]};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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
              {16, 64, 2}, true);
  else       // A[a][s][b]: dims (b, s, a)
    ok = map3(&mA, t.A, {(uint64_t)t.chi_b, 2, (uint64_t)t.chi_a}, {(uint64_t)t.a_s * 8, (uint64_t)t.a_a * 8},
              {16, 2, 64}, true);
  if (ok) {
    if (pfB)   // B[t][b][c]: dims (c, b, t)
      ok = map3(&mB, t.B, {(uint64_t)t.chi_c, (uint64_t)t.chi_b, 2}, {(uint64_t)t.b_b * 8, (uint64_t)t.b_t * 8},
                {8, 16, 1}, false);
    else       // B[b][t][c]: dims (c, t, b)
      ok = map3(&mB, t.B, {(uint64_t)t.chi_c, 2, (uint64_t)t.chi_b}, {(uint64_t)t.b_t * 8, (uint64_t)t.b_b * 8},
                {8, 1, 16}, false);
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
  tebd_tma_kernel<<<(unsigned)((int64_t)a.tiles_m * a.tiles_n), kNT + 32, kSmem, s>>>(mA, mB, a);   // + producer warp
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tci
