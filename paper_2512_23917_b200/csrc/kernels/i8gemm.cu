// i8gemm.cu -- the Ozaki-II residue products on the INT8 tensor cores
// (DESIGN.md §12): one persistent launch computes, for every
// batch plane b of L,
//     D[b][m][n] = (sum_k A[b][m][k] B[b][n][k]) mod m_b      (uint8, in [0, m_b))
// with A [L][M][Kp], B [L][N][Kp] int8 K-major (the residue planes of the two
// operands), exact int32 accumulation (K * 127^2 < 2^31) and the modulus
// m_b = moduli[b / per_mod] of the plane.
//
// Blackwell structure (hand-written tcgen05 / TMA / TMEM, sm_100a):
//  * CTA pairs (cluster 2x1x1) issue tcgen05.mma.cta_group::2.kind::i8 with
//    M = 256 (128 rows per CTA) x N = 256 x K = 32 per instruction; each CTA
//    TMA-loads its 128 rows of A and its 128 rows (half of N) of B for a
//    128-byte K block (SWIZZLE_128B tiles, 32 KB per CTA per stage) and both
//    CTAs' transactions complete on the leader's mbarrier;
//  * warp roles: warp 0 TMA producer, warp 1 MMA issuer (leader CTA; TMEM
//    allocation in both), warps 2-9 epilogue (two per TMEM lane quarter);
//  * accumulators in TMEM (2 x 256 int32 columns: the epilogue of tile i
//    overlaps the main loop of tile i+1), read back with tcgen05.ld 32x32b,
//    reduced mod m_b in integer arithmetic, packed to bytes in shared memory
//    and written by TMA tensor stores (no generic global stores: the
//    release-arrives that hand TMEM back never wait on store traffic);
//  * a dynamic persistent schedule: the leader's producer claims tile ids
//    from a global counter in raster order (plane, then the smaller
//    operand's panels fastest) and broadcasts them to every role of both
//    CTAs through an mbarrier ring, so the tiles in flight always form a
//    compact block of the raster and share their panels in L2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>

#include "../tci_internal.h"
#include "common.cuh"

namespace tci {
namespace i8g {

constexpr int kBM = 128;            // rows of A per CTA (256 per CTA pair)
constexpr int kBN = 256;            // UMMA N (each CTA loads 128 rows of B)
constexpr int kBK = 128;            // bytes of K per stage (4 UMMA K-steps of 32)
constexpr int kStages = 6;
constexpr int kStageBytes = kBM * kBK + (kBN / 2) * kBK;   // 32 KB per CTA
constexpr int kEpiWarps = 8;        // two warps per TMEM lane quarter, 4 column chunks each
constexpr int kThreads = 64 + 32 * kEpiWarps;   // producer, MMA, epilogue warps
constexpr int kTmemCols = 512;      // two 256-column int32 accumulators
constexpr uint32_t kTxBytes = 2u * kStageBytes;             // both CTAs' loads land on the leader's barrier
constexpr int kStgBytes = 2 * 32 * 32;   // per epilogue warp: two 32 x 32-byte output boxes
constexpr size_t kSmemBytes =
    (size_t)kStages * kStageBytes + (size_t)kEpiWarps * kStgBytes + 1024 /* align */ + 512 /* barriers, ids */;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// arrive on the barrier at the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t rank) {
  asm volatile(
      "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
      " mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
// arrival on a barrier of the pair leader (CTA 0): the leader's own threads
// arrive locally (release at CTA scope: a plain SYNCS arrive), the peer's at
// cluster scope (mapa + release.cluster, which ptxas implements with a
// MEMBAR.GPU) -- halves the heavy fences per tile
__device__ __forceinline__ void mbar_arrive_leader(uint64_t *bar, bool leader) {
  if (leader)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
  else
    mbar_arrive_remote(bar, 0);
}
// 3-D TMA load into this CTA's shared memory, completing on the pair leader's
// barrier, with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load_2sm(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2,
                                             uint64_t policy) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;   // peer bit cleared: CTA 0 of the pair
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy(int kind) {
  uint64_t pol;
  if (kind == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  else if (kind == 2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B (8-row x 128-byte
// atoms, 1024 bytes apart), sm_100 descriptor version 1
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: kind::i8, signed A and B, int32 accumulator,
// K-major A and B, M = 256 (cta_group::2), N = 256
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) | ((256u >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(acc)
      : "memory");
}
// completion of this thread's prior tcgen05 ops -> one arrival on `bar` in both CTAs
__device__ __forceinline__ void umma_commit_both(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
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

// x mod m in [0, m) for |x| < 2^31 and odd 64 < m < 256: split
// x = hi 2^16 + lo, y = hi (2^16 mod m) + lo + m 2^16 in [0, 2^25), then
// q = floor(y / m) = umulhi(y, ceil(2^(32+sh) / m)) >> sh with
// sh = floor(log2 m) (the magic fits 32 bits; its excess e < m over
// 2^(32+sh) / m shifts y/m by y e / (m 2^(32+sh)) < 1/m: exact for y < 2^(32+sh) / m)
struct ModM {
  int m, c16, sh;
  uint32_t magic;
  __device__ __forceinline__ void set(int mod) {
    m = mod;
    c16 = 65536 % mod;
    sh = 31 - __clz(mod);
    magic = (uint32_t)(((1ull << (32 + sh)) + (uint64_t)mod - 1) / (uint64_t)mod);
  }
  __device__ __forceinline__ uint32_t operator()(int x) const {
    const uint32_t y = (uint32_t)((x >> 16) * c16 + (x & 0xffff) + (m << 16));
    const uint32_t q = __umulhi(y, magic) >> sh;
    return y - q * (uint32_t)m;
  }
};


struct Params {
  int64_t M, N, Kp;        // rows of A per plane, rows of B (= columns of D), padded K
  int L, per_mod;          // planes, planes per modulus
  int tiles_m, tiles_n;
  int64_t tiles;           // L * tiles_m * tiles_n
  uint8_t *D;              // [L][M][N]
  int *counter;            // dynamic tile counter (zero at launch)
  int a_resident;          // raster: 1 = M tiles fastest (A panels stay in L2), 0 = N tiles fastest
  int res_block;           // resident panels per block of the raster
  int hintA, hintB;        // L2 eviction priority of the A / B loads (0 normal, 1 first, 2 last)
  int mods[16];            // modulus of planes [l * per_mod, (l + 1) * per_mod)
};

// tile index -> (plane, M tile, N tile), planes outermost. Inside a plane one
// operand is "resident": its panels are taken in blocks of res_block (sized
// to stay in L2), and inside a block the resident panel varies fastest while
// the other operand's panels stream by once each. The ~74 tiles in flight
// then share the block's resident panels and a few streamed ones: DRAM reads
// per plane are about (streamed panels x blocks + resident panels).
__device__ __forceinline__ void tile_coords(const Params &p, int64_t t, int &b, int &tm, int &tn) {
  const int64_t per_plane = (int64_t)p.tiles_m * p.tiles_n;
  b = (int)(t / per_plane);
  const int r = (int)(t % per_plane);
  const int nres = p.a_resident ? p.tiles_m : p.tiles_n;   // resident panels
  const int nstr = p.a_resident ? p.tiles_n : p.tiles_m;   // streamed panels
  const int per_block = p.res_block * nstr;
  const int blk = r / per_block, w = r % per_block;
  const int bsz = min(p.res_block, nres - blk * p.res_block);
  const int ir = blk * p.res_block + w % bsz, is = w / bsz;
  tm = p.a_resident ? ir : is;
  tn = p.a_resident ? is : ir;
}

constexpr int kTidSlots = 8;       // depth of the tile-id broadcast ring
constexpr int kTidConsumers = 2 + 2 * kEpiWarps;   // leader: MMA + epilogue warps; peer: producer + epilogue warps

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    i8gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                  const __grid_constant__ CUtensorMap mapD, const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned stage ring (SWIZZLE_128B atoms), barriers behind it
  const uint32_t base_u = smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u + 1023u) & ~1023u) - base_u);
  uint8_t *stg = smem + kStages * kStageBytes;   // epilogue output boxes
  uint64_t *full = reinterpret_cast<uint64_t *>(stg + kEpiWarps * kStgBytes);
  uint64_t *empty = full + kStages;
  uint64_t *tfull = empty + kStages;
  uint64_t *tempty = tfull + 2;
  uint64_t *idfull = tempty + 2;
  uint64_t *idempty = idfull + kTidSlots;
  int *idslot = reinterpret_cast<int *>(idempty + kTidSlots);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(idslot + kTidSlots);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int KB = (int)((p.Kp + kBK - 1) / kBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);   // epilogue warps of both CTAs
    }
    for (int i = 0; i < kTidSlots; i++) {
      mbar_init(&idfull[i], 1);
      mbar_init(&idempty[i], kTidConsumers);
    }
    mbar_fence_init();
  }
  if (warp == 1) {   // TMEM: both CTAs of the pair allocate (cta_group::2)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(tmem_slot);

  // consumer side of the tile-id ring: the next tile of this pair (-1: done)
  int id_i = 0;
  uint32_t id_phase = 0;
  auto next_tile = [&](int &slot) -> int {
    slot = id_i;
    mbar_wait(&idfull[id_i], id_phase);
    const int t = *reinterpret_cast<volatile int *>(&idslot[id_i]);
    if (++id_i == kTidSlots) {
      id_i = 0;
      id_phase ^= 1;
    }
    return t;
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs); the leader's also claims the tile ids =====
    if (lane == 0) {
      const uint64_t polA = l2_policy(p.hintA), polB = l2_policy(p.hintB);
      int stage = 0;
      uint32_t phase = 0;
      int fi = 0;
      uint32_t fphase = 0;
      // leader: publish tile id t in the ring (both CTAs); dynamic schedule:
      // tiles are claimed in raster order as pairs free up, so the tiles in
      // flight stay a compact block of the raster
      auto publish = [&](int t) {
        mbar_wait(&idempty[fi], fphase ^ 1);
        idslot[fi] = t;
        asm volatile(
            "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, 1;\n st.shared::cluster.b32 [ra], %1;\n}\n" ::"r"(
                smem_u32(&idslot[fi])),
            "r"(t)
            : "memory");
        mbar_arrive_remote(&idfull[fi], 0);   // release.cluster: the slot writes are visible first
        mbar_arrive_remote(&idfull[fi], 1);
        if (++fi == kTidSlots) {
          fi = 0;
          fphase ^= 1;
        }
      };
      auto claim = [&]() {
        const int c = atomicAdd(p.counter, 1);
        return c < p.tiles ? c : -1;
      };
      int t;
      if (leader) {
        t = claim();
        publish(t);
      } else {
        int slot;
        t = next_tile(slot);
        mbar_arrive_remote(&idempty[slot], 0);
      }
      while (t >= 0) {
        // the next claim is in flight while this tile's loads issue (its
        // latency stays off the tile boundary)
        const int t_next_raw = leader ? atomicAdd(p.counter, 1) : 0;
        int b, tm, tn;
        tile_coords(p, t, b, tm, tn);
        const int ra = tm * 256 + (int)rank * kBM, rb = tn * kBN + (int)rank * (kBN / 2);
        for (int kb = 0; kb < KB; kb++) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *sa = smem + stage * kStageBytes;
          uint8_t *sb = sa + kBM * kBK;
          if (leader) mbar_expect_tx(&full[stage], kTxBytes);
          tma_load_2sm(sa, &mapA, &full[stage], kb * kBK, ra, b, polA);
          tma_load_2sm(sb, &mapB, &full[stage], kb * kBK, rb, b, polB);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (leader) {
          t = t_next_raw < p.tiles ? t_next_raw : -1;
          publish(t);
        } else {
          int slot;
          t = next_tile(slot);
          mbar_arrive_remote(&idempty[slot], 0);
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA, one thread) =====
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (;;) {
        int slot;
        const int t = next_tile(slot);
        mbar_arrive_leader(&idempty[slot], true);
        if (t < 0) break;
        mbar_wait(&tempty[acc], acc_phase ^ 1);   // both CTAs' epilogues drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * kBN);
        for (int kb = 0; kb < KB; kb++) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kBM * kBK);
#pragma unroll
          for (int k = 0; k < kBK / 32; k++)   // +32 bytes of K = +2 in the descriptor's address field
            umma_i8(d, da + 2 * k, db + 2 * k, (kb | k) != 0);
          umma_commit_both(&empty[stage]);     // frees the stage in both CTAs once these MMAs completed
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_both(&tfull[acc]);         // accumulator ready for both CTAs' epilogues
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===== epilogue: warps 2..9; warp w reads TMEM lane quarter w % 4 and
    // column chunks [4h, 4h + 4) (h = which of the two warps of that quarter) =====
    const int e = warp - 2, q = warp & 3, h = e >> 2;
    uint8_t *box = stg + e * kStgBytes;
    int acc = 0;
    uint32_t acc_phase = 0;
    ModM mod;
    int cur_mod = -1;
    int nbox = 0;
    for (;;) {
      int slot;
      const int t = next_tile(slot);
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&idempty[slot], leader);
      if (t < 0) break;
      int b, tm, tn;
      tile_coords(p, t, b, tm, tn);
      const int mi = b / p.per_mod;
      if (mi != cur_mod) {
        mod.set(p.mods[mi]);
        cur_mod = mi;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row0 = tm * 256 + (int)rank * kBM + q * 32;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kBN);
#pragma unroll 1
      for (int c = 4 * h; c < 4 * h + 4; c++) {
        uint32_t v[32];
        tmem_ld32(taddr + (uint32_t)(c * 32), v);
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; j++)
          w[j] = mod((int)v[4 * j]) | (mod((int)v[4 * j + 1]) << 8) | (mod((int)v[4 * j + 2]) << 16) |
                 (mod((int)v[4 * j + 3]) << 24);
        // 32 rows x 32 bytes through shared memory, out by one TMA store (rows
        // and columns beyond M / N are clipped by the tensor map)
        uint8_t *bx = box + (nbox & 1) * 1024;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        __syncwarp();
        uint4 *dst = reinterpret_cast<uint4 *>(bx + lane * 32);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                           reinterpret_cast<uint64_t>(&mapD)),
                       "r"(tn * kBN + c * 32), "r"(row0), "r"(b), "r"(smem_u32(bx))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        nbox++;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[acc], leader);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kTmemCols)
                 : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// lab overrides (tools/i8gemm_lab.cu): TMA L2 promotion (0 none, 1 128B,
// 2 256B), raster (-1 auto), L2 eviction hints of the A / B loads
int g_i8_promo = 2;
int g_i8_raster = -1;
int g_i8_hintA = 0, g_i8_hintB = 0;
int g_i8_res_mb = 48;   // L2 budget of the resident panels (MB)

// [L][rows][Kp] int8, boxes of 128 bytes x box_rows rows x 1 plane, SWIZZLE_128B
bool make_map(CUtensorMap *m, const void *base, int64_t rows, int64_t Kp, int L, int box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)L};
  const cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)(rows * Kp)};
  const cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapL2promotion promo = g_i8_promo == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                       : g_i8_promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                         : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the output D [L][M][N] uint8 in 32 x 32-byte boxes (TMA stores)
bool make_map_d(CUtensorMap *m, void *base, int64_t M, int64_t N, int L) {
  auto enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)L};
  const cuuint64_t strides[2] = {(cuuint64_t)N, (cuuint64_t)(M * N)};
  const cuuint32_t box[3] = {32, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

}  // namespace i8g

// D[b] = (A[b] B[b]^T) mod m_(b / per_mod) over L planes; A [L][M][Kp],
// B [L][N][Kp] int8 (Kp a multiple of 64, N a multiple of 16), D [L][M][N]
// uint8; counter: one device int of scratch (the dynamic tile counter)
cudaError_t launch_i8gemm(const int8_t *A, const int8_t *B, uint8_t *D, int64_t M, int64_t N, int64_t Kp, int L,
                          int per_mod, const int *moduli, int nmod, int *counter, cudaStream_t s,
                          int64_t *launches) {
  using namespace i8g;
  if (M <= 0 || N <= 0 || L <= 0) return cudaSuccess;
  if (Kp % 64 || N % 16 || (uintptr_t)A % 16 || (uintptr_t)B % 16 || (uintptr_t)D % 16 || !counter)
    return cudaErrorInvalidValue;
  if (!moduli || per_mod < 1 || nmod < 1 || nmod > 16 || (int64_t)per_mod * nmod < L) return cudaErrorInvalidValue;
  for (int l = 0; l < nmod; l++)
    if (moduli[l] <= 64 || moduli[l] >= 256 || !(moduli[l] & 1)) return cudaErrorInvalidValue;
  CUtensorMap ma, mb, md;
  if (!make_map(&ma, A, M, Kp, L, kBM) || !make_map(&mb, B, N, Kp, L, kBN / 2) || !make_map_d(&md, D, M, N, L))
    return cudaErrorNotSupported;
  Params p{};
  p.M = M;
  p.N = N;
  p.Kp = Kp;
  p.L = L;
  p.per_mod = per_mod;
  for (int l = 0; l < 16; l++) p.mods[l] = l < nmod ? moduli[l] : 1;
  p.tiles_m = (int)((M + 255) / 256);
  p.tiles_n = (int)((N + kBN - 1) / kBN);
  p.tiles = (int64_t)L * p.tiles_m * p.tiles_n;
  p.D = D;
  p.counter = counter;
  static const bool env_read = [] {   // tuning overrides: TCI_I8_RES_MB, TCI_I8_RASTER
    if (const char *e = getenv("TCI_I8_RES_MB")) g_i8_res_mb = atoi(e) > 0 ? atoi(e) : g_i8_res_mb;
    if (const char *e = getenv("TCI_I8_RASTER")) g_i8_raster = atoi(e);
    return true;
  }();
  (void)env_read;
  p.a_resident = g_i8_raster >= 0 ? g_i8_raster : (M <= N ? 1 : 0);   // the smaller panel set stays in L2
  {
    const int nres = p.a_resident ? p.tiles_m : p.tiles_n;
    const int64_t fit = ((int64_t)g_i8_res_mb << 20) / (256 * Kp);   // a panel: 256 rows x Kp bytes
    p.res_block = (int)std::max<int64_t>(1, std::min<int64_t>(nres, fit));
  }
  p.hintA = g_i8_hintA;
  p.hintB = g_i8_hintB;
  {
    cudaError_t e = ensure_smem_attr((const void *)i8gemm_kernel, kSmemBytes);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sms();
  const int64_t clusters = std::min<int64_t>(p.tiles, sms / 2);
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  i8gemm_kernel<<<(unsigned)(2 * clusters), kThreads, kSmemBytes, s>>>(ma, mb, md, p);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tci
