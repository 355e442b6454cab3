// crt_mma.cu -- step 3 of the complex Ozaki-II product (Eq. (3) P:213-217 as
// emulated in DESIGN.md §12, Gaussian moduli R33) on the INT8 tensor cores:
// the CRT reconstruction of C' from its 2n residue planes is itself a small
// dense contraction over the planes,
//
//     s[o][j] = sum_k c[k][o] Bd[k][j]          (k < 32 planes, j < 32 digits)
//
// with c[2l] = c+_l = phi+(C') mod m_l, c[2l+1] = c-_l (bytes in [0, m_l)) and
// Bd the base-256 digits of the CRT weights: columns 0..15 the digits of WR_l
// (for both planes of modulus l: Re C' = sum_l (c+_l + c-_l) WR_l mod M),
// columns 16..31 the digits of WI_l (plane c+) and M - WI_l (plane c-:
// Im C' = sum_l (c+_l - c-_l) WI_l mod M). Every s < 30 * 240 * 255 < 2^21 is
// exact in int32 and X = sum_j s[j] 256^j == C' (mod M), 0 <= X < 2n * 240 * M.
//
// Epilogue (per value, exact up to the final rounding; emulated bit for bit in
// tests/test_ozaki_scheme.py): 16-bit digit pairs p_k = s_2k + 256 s_2k+1
// < 2^30 (int32), 32-bit chunks S_c = p_2c + 2^16 p_2c+1 < 2^47 (exact
// doubles), q = rint(X / M) < 2^13 from the top two chunks (|C'| <= M/4,
// R26), R_c = S_c - q M_c exact (M_c the 32-bit chunks of M),
// C' = ((R_3 2^32 + R_2) 2^32 + R_1) 2^32 + R_0 by Horner from the top (the
// first step exact, <= 2 ulp in all), then the 2^(-2t + E_m + E_n) scaling of
// crt_kernel.
//
// Blackwell structure (sm_100a): persistent CTAs, 2 per SM; warp 0 TMA
// producer (SWIZZLE_128B boxes of 128 columns x 32 planes from the plane-major
// residue array -- exactly the MN-major canonical layout of the A operand,
// planes beyond 2n read as zeros), warp 1 issues one tcgen05.mma.kind::i8
// (M = 128 outputs, N = 32 digits, K = 32 planes, unsigned x unsigned -> s32)
// per 128 columns into TMEM (two 128-column accumulators: the epilogue of
// tile i overlaps the MMAs of tile i+1), warps 2..9 read the digit sums with
// tcgen05.ld and run the epilogue: one output per thread per sub-tile, warp
// stores of 32 consecutive complex values. Each CTA takes a contiguous block
// of tiles (row-major), so the guard's row sums flush once per row segment. Compared with crt_kernel (30 x 3
// DFMA chunk sums + unpacking per complex output, FP64 / issue bound) the
// per-output work drops from ~255 to ~110 instructions.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace crtm {

constexpr int kSub = 128;                       // outputs per MMA (TMEM lanes)
constexpr int kSubs = 4;                        // sub-tiles per tile
constexpr int kTW = kSub * kSubs;               // tile: one row x 512 columns
constexpr int kStages = 4;
constexpr int kStageBytes = 32 * kTW;           // 32 planes x 512 columns = 16 KB
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;   // producer, MMA, epilogue warps
constexpr int kTmemCols = 2 * kSubs * 32;       // two accumulators of 4 x 32 columns
constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 1024 /* Bd */ + 1024 /* align */ + 256;

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

// A: MN-major SWIZZLE_128B (128 outputs = one 128-byte atom along M; groups of
// 8 planes 1024 bytes apart = SBO); B: K-major, no swizzle (8 x 16-byte core
// matrices: the two 16-plane halves 128 bytes apart = LBO, groups of 8 digit
// columns 256 bytes apart = SBO); sm_100 descriptor version 1
__device__ __forceinline__ uint64_t desc_a(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(4096 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint64_t desc_b(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
// kind::i8, s32 accumulator, unsigned A and B, A MN-major, B K-major, N = 32, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 15) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// int32 -> double for 0 <= v < 2^31 without the XU pipe: (2^52 + v) - 2^52
__device__ __forceinline__ double u2d(uint32_t v) {
  return __hiloint2double(0x43300000, (int)v) - 4503599627370496.0;
}

// C' from the 16 digit sums of one value (see the header)
template <int NP>
__device__ __forceinline__ double crt_digits(const uint32_t *s, const double (&Mch)[4], double Mtop) {
  constexpr int NC = (NP + 1) / 2;
  double S[NC];
#pragma unroll
  for (int c = 0; c < NC; c++) {
    const uint32_t p0 = s[4 * c] + (s[4 * c + 1] << 8);
    if (2 * c + 1 < NP) {
      const uint32_t p1 = s[4 * c + 2] + (s[4 * c + 3] << 8);
      S[c] = fma(u2d(p1), 65536.0, u2d(p0));
    } else {
      S[c] = u2d(p0);
    }
  }
  // q from the top two chunks (the rest is < 2^80 against M > 2^69: |X/M - q| < 1/4 + 2^-30);
  // Mtop = 2^(32 (NC - 2)) / M
  const double two32 = 4294967296.0;
  const double q = rint(fma(S[NC - 1], two32, S[NC - 2]) * Mtop);
  double r[NC];
#pragma unroll
  for (int j = 0; j < NC; j++) r[j] = fma(-q, Mch[j], S[j]);   // exact: |q M_j| < 2^45
  // C' = sum_j r_j 2^(32 j) by Horner from the top: each partial sum is
  // C' / 2^(32 j) + O(2^15), so every rounding is relative to C' (<= 2 ulp in
  // all; with 4 chunks, M > 2^96, the first step is exact: |.| < 2^47)
  double x = r[NC - 1];
#pragma unroll
  for (int j = NC - 2; j >= 0; j--) x = fma(x, two32, r[j]);
  return x;
}

__device__ __forceinline__ double pow2i(int h) { return h < -1022 ? 0.0 : __hiloint2double((h + 1023) << 20, 0); }
__device__ __forceinline__ void st_c(double2 *p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_c(float2 *p, double2 v) { __stcs(p, make_float2((float)v.x, (float)v.y)); }
// real outputs (float64 / float32 Ozaki GEMMs): the value is v.x
__device__ __forceinline__ void st_c(double *p, double2 v) { __stcs(p, v.x); }
__device__ __forceinline__ void st_c(float *p, double2 v) { __stcs(p, (float)v.x); }

template <int NP, class TO>
__global__ void __launch_bounds__(kThreads, 2)
    crt_mma_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ CrtMmaArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u = smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u + 1023u) & ~1023u) - base_u);   // SWIZZLE_128B atoms: 1024-aligned
  uint8_t *sB = smem + kStages * kStageBytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + 1024);
  uint64_t *empty = full + kStages;
  uint64_t *tfull = empty + kStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tpr = (a.Np + kTW - 1) / kTW;   // tiles per row
  const int64_t ntiles = a.Mc * tpr;
  // blocked schedule: this CTA takes tiles [t_lo, t_hi) in row-major order
  // (consecutive tiles mostly share a row: one guard flush per row segment)
  const int64_t t_lo = ntiles * blockIdx.x / gridDim.x, t_hi = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int64_t r_lo = t_lo / tpr, tr_lo = t_lo % tpr;

  // the digit matrix in the K-major no-swizzle canonical layout:
  // byte (n, k) at (n / 8) 256 + (k / 16) 128 + (n % 8) 16 + k % 16
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    const int k = i >> 5, n = i & 31;
    sB[(n >> 3) * 256 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15)] = a.Bd[k][n];
  }
  fence_proxy_async_smem();   // generic smem writes -> visible to the tensor core (async proxy)
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(tmem_slot);

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t r = r_lo, tr = tr_lo;
      for (int64_t tile = t_lo; tile < t_hi; tile++) {
        const int c0 = (int)tr * kTW;
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], kStageBytes);
        uint8_t *st = smem + stage * kStageBytes;
#pragma unroll
        for (int i = 0; i < kSubs; i++) tma_load(st + i * 4096, &map, &full[stage], c0 + i * kSub, (int)r, 0);
        if (++tr == tpr) {
          tr = 0;
          r++;
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (one thread) =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint64_t db = desc_b(smem_u32(sB));
      for (int64_t tile = t_lo; tile < t_hi; tile++) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * kStageBytes);
#pragma unroll
        for (int i = 0; i < kSubs; i++)
          umma(tmem_base + (uint32_t)(acc * kSubs * 32 + i * 32), desc_a(sa + i * 4096), db);
        umma_commit(&empty[stage]);   // the stage is free once these MMAs read it
        umma_commit(&tfull[acc]);     // the accumulator is ready for the epilogue
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===== epilogue: warp w reads TMEM lane quarter w % 4, sub-tiles {2h, 2h + 1} =====
    // Both sub-tiles are read before any arithmetic and their four values
    // (Re / Im of two outputs) reconstructed in one branch-free block, so the
    // four dependent FP64 chains interleave (the chain latency, not the pipe,
    // bounds a single value).
    const int e = warp - 2, q = warp & 3, h = e >> 2;
    const int ebm = a.rowsq ? *a.eb_max : 0;
    __shared__ double red[2][kEpiWarps];
    int acc = 0;
    uint32_t acc_phase = 0;
    int64_t r = r_lo, tr = tr_lo, tr_first = tr_lo;
    int par = 0;
    double sq = 0.0;
    for (int64_t tile = t_lo; tile < t_hi; tile++) {
      const int64_t m = a.m0 + r;
      const int ea = a.EA[m];
      const int sc0 = -(2 * a.t - ea);
      const int64_t n0 = tr * kTW + 2 * h * kSub + q * 32 + lane, n1 = n0 + kSub;
      const int eb0 = n0 < a.N ? a.EB[n0] : -100000, eb1 = n1 < a.N ? a.EB[n1] : -100000;
      mbar_wait(&tfull[acc], acc_phase);
      __syncwarp();   // tcgen05.ld is .sync.aligned: the warp converged after the spin
      tc_fence_after();
      uint32_t v0[32], v1[32];
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kSubs * 32 + 2 * h * 32);
      tmem_ld32(ta, v0);
      tmem_ld32(ta + 32, v1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);   // TMEM read: hand the accumulator back
      // complex: (Re, Im) of two outputs; real (TO = double / float): columns
      // 0..15 hold the one value's digits, 16..31 are zero
      constexpr bool CPLX = sizeof(TO) == 16 || std::is_same<TO, float2>::value;
      double x[4];
      x[0] = crt_digits<NP>(v0, a.Mch, a.Minv);
      x[2] = crt_digits<NP>(v1, a.Mch, a.Minv);
      if constexpr (CPLX) {
        x[1] = crt_digits<NP>(v0 + 16, a.Mch, a.Minv);
        x[3] = crt_digits<NP>(v1 + 16, a.Mch, a.Minv);
      } else {
        x[1] = x[3] = 0.0;
      }
      // branch-free scaling by 2^sc = 2^h1 2^h2 (h2 = 0, a multiply by 1, whenever
      // 2^sc is a normal double); zero lines (exponent -100000) give exact zeros
      TO *crow = static_cast<TO *>(a.C) + m * a.c_sm;
#pragma unroll
      for (int o = 0; o < 2; o++) {
        const int64_t n = o ? n1 : n0;
        const int eb = o ? eb1 : eb0;
        const bool live = ea > -100000 && eb > -100000;
        const int sc = sc0 + eb;
        // x 2^h1 is exact (x = 0 or an integer >= 1), so the second factor rounds
        // once (subnormal results included; overflow gives inf, as ldexp)
        const int h1 = max(min(sc, 1023), -1022), h2 = min(sc - h1, 1023);
        const double f1 = live ? __hiloint2double((h1 + 1023) << 20, 0) : 0.0, f2 = pow2i(h2);
        const double xr = x[2 * o], xi = x[2 * o + 1];
        const double2 out = make_double2(xr * f1 * f2, xi * f1 * f2);
        if (a.rowsq) {
          const double g = live ? pow2i(-2 * a.t + eb - ebm) : 0.0;
          sq = fma(xr * g, xr * g, sq);
          sq = fma(xi * g, xi * g, sq);
        }
        if (n < a.N) {
          st_c(crow + n, out);
#pragma unroll 1
          for (int pp = 0; pp < a.npeer; pp++) st_c(static_cast<TO *>(a.peer[pp]) + m * a.c_sm + n, out);
        }
      }
      if (a.rowsq) {
        // guard: one slot per row segment of this CTA (the segment's first
        // tile), summed in a fixed order (per-thread tiles ascending, xor tree
        // per warp, warps ascending); the segment's other slots are zeroed
        if (e == 0 && lane == 0 && tr != tr_first) a.rowsq[m * a.slots_per_row + tr] = 0.0;
        if (tr == tpr - 1 || tile == t_hi - 1) {
#pragma unroll
          for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
          if (lane == 0) red[par][e] = sq;
          __syncwarp();
          named_bar_sync(1, 32 * kEpiWarps);
          if (e == 0 && lane == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < kEpiWarps; w++) t += red[par][w];
            a.rowsq[m * a.slots_per_row + tr_first] = t;
          }
          par ^= 1;
          sq = 0.0;
        }
      }
      if (++tr == tpr) {
        tr = 0;
        r++;
        tr_first = 0;
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kTmemCols)
                 : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

template <int NP, class TO>
cudaError_t launch_np(const CUtensorMap &map, const CrtMmaArgs &a, int64_t ntiles, cudaStream_t s) {
  auto kern = crt_mma_kernel<NP, TO>;
  cudaError_t e = ensure_smem_attr((const void *)kern, kSmemBytes);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, 2 * (int64_t)device_sms());   // ntiles >= grid: every CTA has a tile
  kern<<<grid, kThreads, kSmemBytes, s>>>(map, a);
  return cudaGetLastError();
}

}  // namespace crtm

cudaError_t crt_mma_preload() {
  using namespace crtm;
  cudaFuncAttributes fa;
  const void *fns[] = {(const void *)crt_mma_kernel<4, double2>, (const void *)crt_mma_kernel<5, double2>,
                       (const void *)crt_mma_kernel<6, double2>, (const void *)crt_mma_kernel<7, double2>,
                       (const void *)crt_mma_kernel<8, double2>, (const void *)crt_mma_kernel<4, float2>,
                       (const void *)crt_mma_kernel<5, float2>,  (const void *)crt_mma_kernel<6, float2>,
                       (const void *)crt_mma_kernel<7, float2>,  (const void *)crt_mma_kernel<8, float2>,
                       (const void *)crt_mma_kernel<4, double>,  (const void *)crt_mma_kernel<5, double>,
                       (const void *)crt_mma_kernel<6, double>,  (const void *)crt_mma_kernel<7, double>,
                       (const void *)crt_mma_kernel<8, double>,  (const void *)crt_mma_kernel<4, float>,
                       (const void *)crt_mma_kernel<5, float>,   (const void *)crt_mma_kernel<6, float>,
                       (const void *)crt_mma_kernel<7, float>,   (const void *)crt_mma_kernel<8, float>};
  for (const void *f : fns)
    if (cudaError_t e = cudaFuncGetAttributes(&fa, f); e != cudaSuccess) return e;
  return cudaSuccess;
}

int64_t crt_mma_slots_per_row(int64_t Np) { return (Np + crtm::kTW - 1) / crtm::kTW; }

cudaError_t launch_crt_mma(const CrtMmaArgs &a, bool f32_out, bool real, cudaStream_t s) {
  using namespace crtm;
  if (a.Mc <= 0 || a.N <= 0) return cudaSuccess;
  if (a.planes < 1 || a.planes > 32 || a.Np % 16 || (uintptr_t)a.D % 16 || a.nd < 1 || a.nd > 16)
    return cudaErrorInvalidValue;
  auto enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)a.Np, (cuuint64_t)a.Mc, (cuuint64_t)a.planes};
  const cuuint64_t strides[2] = {(cuuint64_t)a.Np, (cuuint64_t)(a.Mc * a.Np)};
  const cuuint32_t box[3] = {(cuuint32_t)kSub, 1, 32};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t *>(a.D), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  const int64_t ntiles = a.Mc * ((a.Np + kTW - 1) / kTW);
  const int np = (a.nd + 1) / 2;   // 16-bit digit pairs
#define TCI_CRT_NP(TO)                                          \
  switch (np) {                                                 \
    case 4: return launch_np<4, TO>(map, a, ntiles, s);         \
    case 5: return launch_np<5, TO>(map, a, ntiles, s);         \
    case 6: return launch_np<6, TO>(map, a, ntiles, s);         \
    case 7: return launch_np<7, TO>(map, a, ntiles, s);         \
    case 8: return launch_np<8, TO>(map, a, ntiles, s);         \
    default: return cudaErrorInvalidValue;                      \
  }
  if (real) {
    if (f32_out) { TCI_CRT_NP(float) }
    TCI_CRT_NP(double)
  }
  if (f32_out) { TCI_CRT_NP(float2) }
  TCI_CRT_NP(double2)
#undef TCI_CRT_NP
}

}  // namespace tci
