// permute.cu -- transpose kernel, Eq. (1) PAPER.md:167-174:
//   out[c_0..c_{n-1}] = in[c'] with c'[perm[k]] = c_k
// Pure data movement: bitwise exact. HBM-bound (roofline = measured copy
// bandwidth, 2 x bytes per element).
//
// The caller (contract.cpp permute_exec / permute_into) has fused adjacent legs that stay adjacent and
// dropped extent-1 legs, so the problem is `n` fused out legs with the input
// stride of each. Two kernels:
//  * copy_rows: the out-fastest leg is also in-contiguous -> each thread
//    moves 16-byte vectors along contiguous runs.
//  * transpose_tiles: the out-fastest leg j is strided in the input and some
//    other leg i is in-contiguous -> a (TI x TJ) tile is read along i with
//    16-byte loads into padded shared memory and written along j with
//    16-byte stores; every other leg indexes the tile grid.
#include <algorithm>
#include <cstdlib>

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

struct FDiv {                  // n / d for n < 2^31 (Granlund-Montgomery)
  uint32_t d, m;
  int s;                       // shift, -1 for d == 1
};
inline FDiv make_fdiv(uint32_t d) {
  FDiv f{d, 0, -1};
  if (d <= 1) return f;
  int l = 0;
  while ((1ull << l) < d) l++;
  const int p = 31 + l;
  f.m = (uint32_t)(((1ull << p) + d - 1) / d);
  f.s = p - 32;
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FDiv &f) { return f.s < 0 ? n : __umulhi(n, f.m) >> f.s; }

struct RowArgs {
  int nb;
  int64_t bshape[kMaxOrder];
  int64_t b_in[kMaxOrder];
  FDiv bdiv[kMaxOrder];  // 32-bit division by bshape (used when rows * vec_per_row < 2^31)
  FDiv vdiv;             // ... and by vec_per_row
  int64_t run;          // contiguous run length (elements), out rows are contiguous
  int64_t rows;
  int64_t vec_per_row;
  const char *in;
  char *out;
};

// Each thread moves U vectors per pass (all loads issued before the stores:
// memory-level parallelism), coordinates by 32-bit invariant division when
// the vector count fits (64-bit division costs ~40 instructions per leg).
template <int ESZ, int VEC, bool SMALL>
__global__ void __launch_bounds__(256) copy_rows(const __grid_constant__ RowArgs a) {
  using E = typename std::conditional<ESZ == 16, int4,
                                      typename std::conditional<ESZ == 8, int2, int>::type>::type;
  using V = typename std::conditional<
      ESZ * VEC == 16, int4,
      typename std::conditional<ESZ * VEC == 8, int2, int>::type>::type;
  constexpr int U = 4;
  const int64_t total = a.rows * a.vec_per_row;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const E *__restrict__ inE = reinterpret_cast<const E *>(a.in);
  E *__restrict__ outE = reinterpret_cast<E *>(a.out);
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < total; base += U * stride) {
    V val[U];
    int64_t dst_off[U];
    bool full[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t idx = base + u * stride;
      dst_off[u] = -1;
      if (idx >= total) continue;
      int64_t row, v, in_off = 0;
      if (SMALL) {
        uint32_t r32 = fdiv((uint32_t)idx, a.vdiv);
        v = (uint32_t)idx - r32 * a.vdiv.d;
        row = r32;
        for (int k = a.nb - 1; k >= 0; k--) {
          const uint32_t q = fdiv(r32, a.bdiv[k]);
          in_off += (int64_t)(r32 - q * a.bdiv[k].d) * a.b_in[k];
          r32 = q;
        }
      } else {
        row = idx / a.vec_per_row;
        v = idx % a.vec_per_row;
        int64_t r = row;
        for (int k = a.nb - 1; k >= 0; k--) {
          const int64_t c = r % a.bshape[k];
          r /= a.bshape[k];
          in_off += c * a.b_in[k];
        }
      }
      const E *src = inE + in_off + v * VEC;
      dst_off[u] = row * a.run + v * VEC;
      full[u] = VEC > 1 && (v + 1) * VEC <= a.run;
      if (full[u]) {
        val[u] = __ldg(reinterpret_cast<const V *>(src));
      } else {
        E *ve = reinterpret_cast<E *>(&val[u]);
        for (int e = 0; e < VEC; e++) ve[e] = v * VEC + e < a.run ? src[e] : E{};
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (dst_off[u] < 0) continue;
      E *dst = outE + dst_off[u];
      if (full[u]) {
        *reinterpret_cast<V *>(dst) = val[u];
      } else {
        const E *ve = reinterpret_cast<const E *>(&val[u]);
        const int64_t v0 = dst_off[u] % a.run;
        for (int e = 0; e < VEC && v0 + e < a.run; e++) dst[e] = ve[e];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Leg-group tiles (general case). The tile is the product of a group G of
// legs: the input-fastest legs (a contiguous input block of >= RUN elements)
// and the output-fastest legs (a contiguous output block of >= RUN elements);
// at most one leg of each run is cut into chunks. Every other leg (and the
// chunk index of a cut leg) indexes the tiles. A CTA stages one tile in
// shared memory: the load phase walks the tile in input order (contiguous
// runs of Pi elements), the store phase in output order (runs of Po); the
// in-tile coordinates come from 32-bit division by invariant integers.
// Persistent CTAs loop over the tiles.
// ---------------------------------------------------------------------------
constexpr int kGMax = 8;

struct GroupArgs {
  int ng;                                  // legs in the tile
  int TS;                                  // tile elements
  // tile legs in INPUT order (fastest first): extent in the tile, strides,
  // shared-memory stride (tile stored in input order), full extent and cut flag
  FDiv gi_div[kGMax];
  int64_t gi_in[kGMax], gi_out[kGMax];
  int gi_cut[kGMax];                       // index into the cut arrays, or -1
  // the same legs in OUTPUT order
  FDiv go_div[kGMax];
  int64_t go_out[kGMax];
  int go_sm[kGMax];
  int go_cut[kGMax];
  // cut legs (<= 2): full extent; their chunk coordinate comes from the tile index;
  // in-tile coordinate of cut leg c at input position q: (q / ci_pre[c]) % ci_ext[c]
  // (and at output position p with co_pre)
  int ncut;
  int64_t cut_ext[2];
  FDiv ci_pre[2], co_pre[2], c_ext[2];
  // tile-grid legs (outer legs + chunk indices of cut legs), slowest first
  int nb;
  int64_t b_ext[2 * kMaxOrder], b_in[2 * kMaxOrder], b_out[2 * kMaxOrder];
  int b_cut[2 * kMaxOrder];                // cut index when the grid leg is a chunk index, else -1
  int64_t b_chunk[2 * kMaxOrder];          // chunk length for chunk-index legs
  FDiv b_div[2 * kMaxOrder];               // division by b_ext (ntiles < 2^31)
  int64_t ntiles;
  const char *in;
  char *out;
};

// Shared-memory slot of tile position x: XOR-swizzled within blocks of
// W = 128 / ESZ elements (one 128-byte wavefront) by a hash of the higher
// bits, so both the input-order writes (consecutive x) and the output-order
// reads (x strided by any power of two) are free of bank conflicts.
template <int ESZ>
__device__ __forceinline__ int swz(int x) {
  constexpr int W = 128 / ESZ, B = W == 32 ? 5 : (W == 16 ? 4 : 3);
  return x ^ (((x >> B) ^ (x >> (2 * B)) ^ (x >> (3 * B))) & (W - 1));
}

// V elements per vector (16 / 8 / 4-byte accesses): the tile's input-fastest
// and output-fastest legs both hold whole vectors (planner check), so the
// full-tile path moves V consecutive elements per global access.
template <int ESZ, int V>
__global__ void __launch_bounds__(256) permute_groups(const __grid_constant__ GroupArgs a) {
  constexpr int GU = ESZ * V >= 16 ? 4 : 8;
  using E = typename std::conditional<ESZ == 16, int4,
                                      typename std::conditional<ESZ == 8, int2, int>::type>::type;
  using VT = typename std::conditional<
      ESZ * V == 16, int4, typename std::conditional<ESZ * V == 8, int2, int>::type>::type;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int TS = a.TS;
  constexpr int W = 128 / ESZ;
  const int TSP = (TS + W - 1) / W * W;                                // swizzle blocks are whole
  E *tile = reinterpret_cast<E *>(smraw);
  int32_t *ld_off = reinterpret_cast<int32_t *>(tile + TSP);          // in offset of tile position q
  int32_t *st_off = ld_off + TS;                                      // out offset of output position p
  uint16_t *st_slot = reinterpret_cast<uint16_t *>(st_off + TS);      // smem slot of p
  const E *in = reinterpret_cast<const E *>(a.in);
  E *out = reinterpret_cast<E *>(a.out);
  // offset tables of the tile geometry, built once per CTA (full tiles)
  for (int q = threadIdx.x; q < TS; q += 256) {
    uint32_t r = (uint32_t)q;
    int64_t off = 0;
#pragma unroll
    for (int l = 0; l < kGMax; l++) {
      if (l < a.ng) {
        const uint32_t nq = fdiv(r, a.gi_div[l]);
        off += (int64_t)(r - nq * a.gi_div[l].d) * a.gi_in[l];
        r = nq;
      }
    }
    ld_off[q] = (int32_t)off;
    r = (uint32_t)q;
    off = 0;
    int slot = 0;
#pragma unroll
    for (int l = 0; l < kGMax; l++) {
      if (l < a.ng) {
        const uint32_t nq = fdiv(r, a.go_div[l]);
        const uint32_t c = r - nq * a.go_div[l].d;
        r = nq;
        off += (int64_t)c * a.go_out[l];
        slot += (int)c * a.go_sm[l];
      }
    }
    st_off[q] = (int32_t)off;
    st_slot[q] = (uint16_t)swz<ESZ>(slot);
  }
  __syncthreads();
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    uint32_t rem = (uint32_t)t;
    int64_t in_base = 0, out_base = 0;
    int64_t cut_base[2] = {0, 0};
    bool full = true;
    for (int k = a.nb - 1; k >= 0; k--) {
      const uint32_t qk = fdiv(rem, a.b_div[k]);
      const int64_t c = rem - qk * a.b_div[k].d;
      rem = qk;
      in_base += c * a.b_in[k];
      out_base += c * a.b_out[k];
      if (a.b_cut[k] >= 0) {
        cut_base[a.b_cut[k]] = c * a.b_chunk[k];
        full = full && (c * a.b_chunk[k] + a.b_chunk[k] <= a.cut_ext[a.b_cut[k]]);
      }
    }
    if (full) {
      // GU vector loads in flight per thread before their shared-memory stores
      const int TV = TS / V;
      for (int i0 = threadIdx.x; i0 < TV; i0 += 256 * GU) {
        VT v[GU];
#pragma unroll
        for (int u = 0; u < GU; u++) {
          const int i = i0 + u * 256;
          if (i < TV) v[u] = __ldg(reinterpret_cast<const VT *>(in + in_base + ld_off[i * V]));
        }
#pragma unroll
        for (int u = 0; u < GU; u++) {
          const int i = i0 + u * 256;
          if (i < TV) {
            const E *ve = reinterpret_cast<const E *>(&v[u]);
            const int sq = swz<ESZ>(i * V);     // V | W: the vector stays in one swizzle block
#pragma unroll
            for (int e = 0; e < V; e++) tile[sq ^ e] = ve[e];
          }
        }
      }
      __syncthreads();
#pragma unroll 4
      for (int i = threadIdx.x; i < TV; i += 256) {
        VT v;
        E *ve = reinterpret_cast<E *>(&v);
#pragma unroll
        for (int e = 0; e < V; e++) ve[e] = tile[st_slot[i * V + e]];
        *reinterpret_cast<VT *>(out + out_base + st_off[i * V]) = v;
      }
      __syncthreads();
      continue;
    }
    // ragged chunk of a cut leg: bounds from the cut legs' coordinates
    for (int q = threadIdx.x; q < TS; q += 256) {
      bool ok = true;
      for (int c = 0; c < a.ncut; c++) {
        const uint32_t x = fdiv((uint32_t)q, a.ci_pre[c]);
        ok = ok && (cut_base[c] + (x - fdiv(x, a.c_ext[c]) * a.c_ext[c].d) < a.cut_ext[c]);
      }
      if (ok) tile[swz<ESZ>(q)] = in[in_base + ld_off[q]];
    }
    __syncthreads();
    for (int p = threadIdx.x; p < TS; p += 256) {
      bool ok = true;
      for (int c = 0; c < a.ncut; c++) {
        const uint32_t x = fdiv((uint32_t)p, a.co_pre[c]);
        ok = ok && (cut_base[c] + (x - fdiv(x, a.c_ext[c]) * a.c_ext[c].d) < a.cut_ext[c]);
      }
      if (ok) out[out_base + st_off[p]] = tile[st_slot[p]];
    }
    __syncthreads();
  }
}

// Plan the leg-group tile; false when it does not apply (caller falls back).
template <int ESZ>
bool plan_groups(const PermuteProblem &p, const int64_t *out_stride, GroupArgs &a) {
  const int n = p.n;
  // >= 256 contiguous bytes per run; 16 KB tiles, 8 CTAs per SM (measured
  // against 8/24/32/64 KB tiles and 512/1024-byte runs: tools/gpu_perm_sweep.sh)
  constexpr int RUN = 256 / ESZ;
  constexpr int TSMAX = 16384 / ESZ;
  int ord_in[kMaxOrder], ord_out[kMaxOrder];
  for (int k = 0; k < n; k++) ord_in[k] = ord_out[k] = k;
  std::sort(ord_in, ord_in + n, [&](int x, int y) { return p.in_stride_for_out[x] < p.in_stride_for_out[y]; });
  std::sort(ord_out, ord_out + n, [&](int x, int y) { return out_stride[x] < out_stride[y]; });
  int64_t tex[kMaxOrder];                    // tile extent per leg (0 = not in the tile)
  for (int k = 0; k < n; k++) tex[k] = 0;
  int cut_leg[2] = {-1, -1}, ncut = 0;
  int64_t TS = 1;
  auto add_run = [&](const int *ord, int64_t target) {
    int64_t run = 1;
    for (int i = 0; i < n && run < target; i++) {
      const int k = ord[i];
      const int64_t e = p.shape_out[k];
      if (tex[k] > 0) {                      // already in the tile
        run *= tex[k];
        if (tex[k] < e) break;               // a cut leg ends the contiguous run
        continue;
      }
      const int64_t room = TSMAX / TS;
      if (room < 2) break;
      if (e <= room && (run * e <= 4 * target || e <= 2)) {
        tex[k] = e;
        TS *= e;
        run *= e;
      } else {                               // cut into chunks
        int64_t ch = std::min<int64_t>(room, std::max<int64_t>(2, (target + run - 1) / run));
        ch = std::min(ch, e);
        if (ch < e) ch = (e + (e + ch - 1) / ch - 1) / ((e + ch - 1) / ch);   // balanced: no sliver chunk
        tex[k] = ch;
        TS *= ch;
        run *= ch;
        if (ch < e) cut_leg[ncut++] = k;
        break;
      }
    }
  };
  add_run(ord_in, RUN);
  add_run(ord_out, RUN);
  // grow the tile towards TSMAX: widen the cut legs first (input-run cut
  // first), then take further legs in input order
  for (int c = 0; c < ncut; c++) {
    const int k = cut_leg[c];
    const int64_t e = p.shape_out[k];
    const int64_t grow = std::min<int64_t>(TSMAX / TS, (e + tex[k] - 1) / tex[k]);
    if (grow >= 2) {
      TS = TS / tex[k];
      // balanced chunks: the last one is not a sliver
      const int64_t cmax = std::min<int64_t>(e, tex[k] * grow), nch = (e + cmax - 1) / cmax;
      tex[k] = (e + nch - 1) / nch;
      TS *= tex[k];
    }
  }
  for (int i = 0; i < n && 2 * TS <= TSMAX; i++) {
    const int k = ord_in[i];
    if (tex[k] > 0) continue;
    const int64_t e = p.shape_out[k], room = TSMAX / TS;
    if (e <= room) {
      tex[k] = e;
      TS *= e;
    } else if (ncut < 2) {
      tex[k] = room;
      TS *= room;
      cut_leg[ncut++] = k;
    }
    break;   // one extra leg at most: keep the tile's leg count small
  }
  // a cut leg that grew to its full extent is no longer cut
  for (int c = 0; c < ncut; c++)
    if (tex[cut_leg[c]] >= p.shape_out[cut_leg[c]]) {
      cut_leg[c] = cut_leg[ncut - 1];
      cut_leg[ncut - 1] = -1;
      ncut--;
      c--;
    }
  int ng = 0;
  for (int k = 0; k < n; k++) ng += tex[k] > 0;
  if (ng > kGMax || TS < 2 || p.total >= (int64_t(1) << 31)) return false;   // int32 in-tile offsets
  a.ng = ng;
  a.TS = (int)TS;
  a.ncut = ncut;
  // legs in input order with their smem strides (tile stored in input order)
  int64_t sm_of[kMaxOrder];
  {
    int l = 0;
    int64_t sm = 1;
    for (int i = 0; i < n; i++) {
      const int k = ord_in[i];
      if (!tex[k]) continue;
      a.gi_div[l] = make_fdiv((uint32_t)tex[k]);
      a.gi_in[l] = p.in_stride_for_out[k];
      a.gi_out[l] = out_stride[k];
      a.gi_cut[l] = k == cut_leg[0] ? 0 : (k == cut_leg[1] ? 1 : -1);
      sm_of[k] = sm;
      sm *= tex[k];
      l++;
    }
    l = 0;
    for (int i = 0; i < n; i++) {
      const int k = ord_out[i];
      if (!tex[k]) continue;
      a.go_div[l] = make_fdiv((uint32_t)tex[k]);
      a.go_out[l] = out_stride[k];
      a.go_sm[l] = (int)sm_of[k];
      a.go_cut[l] = k == cut_leg[0] ? 0 : (k == cut_leg[1] ? 1 : -1);
      l++;
    }
  }
  for (int c = 0; c < 2; c++) {
    a.cut_ext[c] = c < ncut ? p.shape_out[cut_leg[c]] : 0;
    a.c_ext[c] = make_fdiv(c < ncut ? (uint32_t)tex[cut_leg[c]] : 1u);
    int64_t pi = 1, po = 1;
    for (int i = 0; c < ncut && i < n; i++) {
      const int k = ord_in[i];
      if (k == cut_leg[c]) break;
      if (tex[k]) pi *= tex[k];
    }
    for (int i = 0; c < ncut && i < n; i++) {
      const int k = ord_out[i];
      if (k == cut_leg[c]) break;
      if (tex[k]) po *= tex[k];
    }
    a.ci_pre[c] = make_fdiv((uint32_t)pi);
    a.co_pre[c] = make_fdiv((uint32_t)po);
  }
  // tile grid: legs outside the tile and chunk indices of cut legs (output order, slowest first)
  a.nb = 0;
  a.ntiles = 1;
  for (int k = 0; k < n; k++) {
    if (tex[k] == 0) {
      a.b_ext[a.nb] = p.shape_out[k];
      a.b_in[a.nb] = p.in_stride_for_out[k];
      a.b_out[a.nb] = out_stride[k];
      a.b_cut[a.nb] = -1;
      a.b_chunk[a.nb] = 0;
    } else if (tex[k] < p.shape_out[k]) {
      const int64_t ch = tex[k];
      a.b_ext[a.nb] = (p.shape_out[k] + ch - 1) / ch;
      a.b_in[a.nb] = ch * p.in_stride_for_out[k];
      a.b_out[a.nb] = ch * out_stride[k];
      a.b_cut[a.nb] = k == cut_leg[0] ? 0 : 1;
      a.b_chunk[a.nb] = ch;
    } else {
      continue;
    }
    a.ntiles *= a.b_ext[a.nb];
    a.b_div[a.nb] = make_fdiv((uint32_t)std::min<int64_t>(a.b_ext[a.nb], 0x7fffffff));
    a.nb++;
  }
  if (a.ntiles >= (int64_t(1) << 31)) return false;
  a.in = static_cast<const char *>(p.in);
  a.out = static_cast<char *>(p.out);
  return true;
}

// Small tensors (<= 8 MB, L2-resident): one output element per thread in
// output order (coalesced stores), its input offset from the output index by
// multiply-high divisions, reads served by L2. The tiled kernels' per-CTA
// setup (offset tables, tile geometry) is the cost at this size: a 2 MB
// six-leg permute took ~28 us through the leg-group tiles.
constexpr int64_t kSmallPermuteBytes = 8 << 20;
// TCI_PERMUTE_SMALL=0 sends small tensors through the tiled kernels (A/B)
bool small_permute_disabled() {
  static const bool off = [] {
    const char *e = getenv("TCI_PERMUTE_SMALL");
    return e && e[0] == '0';
  }();
  return off;
}
struct SmallArgs {
  int n;
  FDiv div[kMaxOrder];      // output extents, fastest first
  int64_t in_st[kMaxOrder]; // input strides, fastest first
  int64_t total;
  const void *in;
  void *out;
};
template <int ESZ>
__global__ void __launch_bounds__(256) permute_small(const __grid_constant__ SmallArgs a) {
  using E = typename std::conditional<ESZ == 16, int4,
                                      typename std::conditional<ESZ == 8, int2, int>::type>::type;
  const E *in = reinterpret_cast<const E *>(a.in);
  E *out = reinterpret_cast<E *>(a.out);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.total; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r = (uint32_t)i;
    int64_t off = 0;
#pragma unroll 4
    for (int k = 0; k < a.n; k++) {
      const uint32_t q = fdiv(r, a.div[k]);
      off += (int64_t)(r - q * a.div[k].d) * a.in_st[k];
      r = q;
    }
    out[i] = __ldg(in + off);
  }
}

template <int ESZ>
cudaError_t launch_typed(const PermuteProblem &p, cudaStream_t s, int64_t *launches) {
  const int n = p.n;
  if (n > 1 && p.total * ESZ <= kSmallPermuteBytes && p.total < (1LL << 31) && !small_permute_disabled()) {
    SmallArgs a{};
    a.n = n;
    a.total = p.total;
    a.in = p.in;
    a.out = p.out;
    for (int k = 0; k < n; k++) {
      a.div[k] = make_fdiv((uint32_t)p.shape_out[n - 1 - k]);
      a.in_st[k] = p.in_stride_for_out[n - 1 - k];
    }
    const int64_t blocks = std::min<int64_t>((p.total + 255) / 256, 148 * 8);
    permute_small<ESZ><<<(unsigned)blocks, 256, 0, s>>>(a);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  int64_t out_stride[kMaxOrder];
  {
    int64_t st = 1;
    for (int k = n - 1; k >= 0; k--) { out_stride[k] = st; st *= p.shape_out[k]; }
  }
  constexpr int VMAX = 16 / ESZ;
  auto aligned = [&](const void *ptr) { return ((uintptr_t)ptr % 16) == 0; };
  // contiguous runs: vectorised row copies when the runs are >= 128 bytes and
  // 16-byte aligned (odd runs go to the leg-group tiles)
  bool rows_vec = n > 0 && p.in_stride_for_out[n - 1] == 1 && aligned(p.in) && aligned(p.out) &&
                  p.shape_out[n - 1] % VMAX == 0;
  for (int k = 0; rows_vec && k < n - 1; k++) rows_vec = p.in_stride_for_out[k] % VMAX == 0;
  auto rows_path = [&]() -> cudaError_t {
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
    const bool small = total < (int64_t(1) << 31);
    if (small) {
      a.vdiv = make_fdiv((uint32_t)a.vec_per_row);
      for (int k = 0; k < a.nb; k++) a.bdiv[k] = make_fdiv((uint32_t)a.bshape[k]);
    }
    // 4 vectors per thread per pass; 8 CTAs of 256 per SM
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + 1023) / 1024, 148 * 8));
    if (vec_ok) {
      if (small) copy_rows<ESZ, VMAX, true><<<(unsigned)blocks, 256, 0, s>>>(a);
      else copy_rows<ESZ, VMAX, false><<<(unsigned)blocks, 256, 0, s>>>(a);
    } else {
      if (small) copy_rows<ESZ, 1, true><<<(unsigned)blocks, 256, 0, s>>>(a);
      else copy_rows<ESZ, 1, false><<<(unsigned)blocks, 256, 0, s>>>(a);
    }
    if (launches) ++*launches;
    return cudaGetLastError();
  };
  const bool in_run = n > 0 && p.in_stride_for_out[n - 1] == 1;
  // row copies for contiguous runs >= 512 B; shorter runs go to leg-group tiles,
  // which also group the writes (128-byte runs: 0.81 -> 0.87 of a plain copy)
  if (n <= 1 || (in_run && p.shape_out[n - 1] * ESZ >= 512 && rows_vec)) return rows_path();
  // tile legs of the classic transpose: j = out-fastest leg, i = the
  // in-contiguous leg; when both are long it is the fastest kernel
  constexpr int T = (ESZ == 16) ? 32 : 64;
  int li = -1;
  for (int k = 0; k < n - 1; k++)
    if (p.in_stride_for_out[k] == 1) li = k;
  // (both legs at least one full tile: a half-empty tile wastes half the CTA)
  const bool classic = li >= 0 && p.shape_out[li] >= T && p.shape_out[n - 1] >= T;
  // otherwise leg-group tiles (short contiguous legs are grouped until both
  // the reads and the writes move >= 256 contiguous bytes)
  if (!classic) {
    GroupArgs ga;
    if (plan_groups<ESZ>(p, out_stride, ga)) {
      constexpr int W = 128 / ESZ;
      const size_t smem = (size_t)((ga.TS + W - 1) / W * W) * ESZ + (size_t)ga.TS * 10 + 16;
      // vectors: V consecutive elements along the tile's input-fastest leg
      // (unit input stride) and its output-fastest leg (unit output stride);
      // every other stride and chunk base a multiple of V, 16-byte bases
      int V = VMAX;
      auto vec_ok = [&](int v) {
        if (v == 1) return true;
        if ((uintptr_t)p.in % (v * ESZ) || (uintptr_t)p.out % (v * ESZ)) return false;
        if (ga.gi_in[0] != 1 || ga.gi_div[0].d % v || ga.go_out[0] != 1 || ga.go_div[0].d % v) return false;
        for (int l = 1; l < ga.ng; l++) if (ga.gi_in[l] % v) return false;
        for (int l = 1; l < ga.ng; l++) if (ga.go_out[l] % v) return false;
        for (int k = 0; k < ga.nb; k++) if (ga.b_in[k] % v || ga.b_out[k] % v) return false;
        return ga.TS % v == 0;
      };
      while (V > 1 && !vec_ok(V)) V /= 2;
      auto k = permute_groups<ESZ, 1>;
      if (V == 4) k = permute_groups<ESZ, (VMAX >= 4 ? 4 : 1)>;
      else if (V == 2) k = permute_groups<ESZ, (VMAX >= 2 ? 2 : 1)>;
      cudaError_t e = ensure_smem_attr((const void *)k, smem);
      if (e != cudaSuccess) return e;
      const int64_t blocks = std::min<int64_t>(ga.ntiles, 148 * 8);
      k<<<(unsigned)blocks, 256, smem, s>>>(ga);
      if (launches) ++*launches;
      return cudaGetLastError();
    }
  }
  if (in_run || li < 0) return rows_path();   // no leg-group plan: plain row copies
  // tile transpose between j = out-fastest leg and i = the in-contiguous leg
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

namespace {
struct OffLegs {
  int nl;
  int64_t ext[kMaxOrder], stride[kMaxOrder];
};
__global__ void offsets_kernel(int64_t *offs, int64_t n, const OffLegs L) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i, o = 0;
    for (int l = L.nl - 1; l >= 0; l--) {
      o += (r % L.ext[l]) * L.stride[l];
      r /= L.ext[l];
    }
    offs[i] = o;
  }
}
// both tables of a scatter epilogue in one launch: index i < n1 fills offs1
// from L1, the rest offs2 from L2
__global__ void offsets2_kernel(int64_t *offs1, int64_t n1, const OffLegs L1, int64_t *offs2, int64_t n2,
                                const OffLegs L2) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n1 + n2; j += (int64_t)gridDim.x * blockDim.x) {
    const bool first = j < n1;
    const OffLegs &L = first ? L1 : L2;
    const int64_t i = first ? j : j - n1;
    int64_t r = i, o = 0;
    for (int l = L.nl - 1; l >= 0; l--) {
      o += (r % L.ext[l]) * L.stride[l];
      r /= L.ext[l];
    }
    (first ? offs1 : offs2)[i] = o;
  }
}
}  // namespace

cudaError_t launch_offsets2(int64_t *offs1, int64_t n1, int nl1, const int64_t *ext1, const int64_t *stride1,
                            int64_t *offs2, int64_t n2, int nl2, const int64_t *ext2, const int64_t *stride2,
                            cudaStream_t s, int64_t *launches) {
  if (n1 + n2 == 0) return cudaSuccess;
  if (nl1 > kMaxOrder || nl2 > kMaxOrder) return cudaErrorInvalidValue;
  OffLegs L1{}, L2{};
  L1.nl = nl1;
  L2.nl = nl2;
  for (int l = 0; l < nl1; l++) { L1.ext[l] = ext1[l]; L1.stride[l] = stride1[l]; }
  for (int l = 0; l < nl2; l++) { L2.ext[l] = ext2[l]; L2.stride[l] = stride2[l]; }
  offsets2_kernel<<<(unsigned)std::min<int64_t>((n1 + n2 + 255) / 256, 148 * 4), 256, 0, s>>>(offs1, n1, L1, offs2,
                                                                                           n2, L2);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_offsets(int64_t *offs, int64_t n, int nl, const int64_t *ext, const int64_t *stride,
                           cudaStream_t s, int64_t *launches) {
  if (n == 0) return cudaSuccess;
  if (nl > kMaxOrder) return cudaErrorInvalidValue;
  OffLegs L{};
  L.nl = nl;
  for (int l = 0; l < nl; l++) {
    L.ext[l] = ext[l];
    L.stride[l] = stride[l];
  }
  offsets_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4), 256, 0, s>>>(offs, n, L);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_copy(void *dst, const void *src, size_t bytes, cudaStream_t s, int64_t *launches) {
  (void)launches;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s);
}

}  // namespace tci
