// svd.cu -- the matrix SVD under tci::svd / tci::trunc_svd (
// SURVEY 8(f2)): block one-sided (Hestenes) Jacobi on the FP64 tensor cores.
//
// The matricized A' (I x J) is held as X = A' (I <= J) or
// X = A'^H (I > J): n = min(I, J) rows of length L = max(I, J), padded with
// zero rows to a multiple of 32. Rows are grouped in blocks of SB = 16; a
// sweep pairs every two blocks once (round-robin, nb - 1 rounds of nb/2
// disjoint pairs). One CTA handles one block pair per round:
//   1. Gram   H = X_p X_p^H  (32 x 32 Hermitian, DMMA m8n8k4, k split over
//              the 8 warps, partials added in warp order -> deterministic);
//   2. test   max_{i<j} |H_ij| / sqrt(H_ii H_jj) <= tol -> pair converged,
//              nothing is written (the sweep maximum goes to *offmax);
//   3. eig    H = G diag(ev) G^H by parallel cyclic Jacobi in shared memory
//              (16 disjoint 2x2 rotations per step, blockwise J^H H J);
//   4. update X_p <- G^H X_p and Y_p <- G^H Y_p (DMMA, in place).
// Converged rows are x_i = s_i v_i^H (X = Q A') with Q = Y accumulated from
// Y0 = I, so A' = Q^H diag(s) V^H: singular values are row norms, one factor
// is Y, the other the normalized rows. Every reduction has a fixed order, so
// results are bitwise reproducible.
#include <cfloat>
#include <cmath>

#include <cooperative_groups.h>

#include "../tci_internal.h"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace tci {
namespace {

constexpr int SB = 16;       // rows per block
constexpr int PR = 2 * SB;   // rows per block pair (one cluster of CTAs)
constexpr int NT = 256;      // threads per CTA (8 warps)
constexpr int HP = PR + 1;   // pitch of H and G in shared memory

template <bool C> struct Cx;
template <> struct Cx<false> {
  using E = double;
  static constexpr int CW = 64;          // columns per staged chunk
  static constexpr int NST = 4;          // cp.async stages
  static constexpr int PITCH = CW + 4;   // conflict-free fragment loads (8-byte banks)
  static constexpr int PER16 = 2;        // elements per 16-byte copy
};
template <> struct Cx<true> {
  using E = double2;
  static constexpr int CW = 32;
  static constexpr int NST = 4;
  static constexpr int PITCH = CW + 2;
  static constexpr int PER16 = 1;
};

__device__ __forceinline__ double re(double x) { return x; }
__device__ __forceinline__ double re(double2 x) { return x.x; }
__device__ __forceinline__ double cabs(double x) { return fabs(x); }
__device__ __forceinline__ double cabs(double2 x) { return hypot(x.x, x.y); }
__device__ __forceinline__ double abs2(double x) { return x * x; }
__device__ __forceinline__ double abs2(double2 x) { return fma(x.x, x.x, x.y * x.y); }
__device__ __forceinline__ double cj(double x) { return x; }
__device__ __forceinline__ double2 cj(double2 x) { return make_double2(x.x, -x.y); }
__device__ __forceinline__ double cmul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double cadd(double a, double b) { return a + b; }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double rmul(double s, double a) { return s * a; }
__device__ __forceinline__ double2 rmul(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
template <class E> __device__ __forceinline__ E czero();
template <> __device__ __forceinline__ double czero<double>() { return 0.0; }
template <> __device__ __forceinline__ double2 czero<double2>() { return make_double2(0.0, 0.0); }
template <class E> __device__ __forceinline__ E cone();
template <> __device__ __forceinline__ double cone<double>() { return 1.0; }
template <> __device__ __forceinline__ double2 cone<double2>() { return make_double2(1.0, 0.0); }
__device__ __forceinline__ double phase_of(double h, double ah) { return h >= 0.0 ? 1.0 : -1.0; }   // conj(h)/|h|
__device__ __forceinline__ double2 phase_of(double2 h, double ah) {
  return make_double2(h.x / ah, -h.y / ah);   // (not h * (1/ah): 1/ah overflows for subnormal |h|)
}

// A row whose squared norm is below 1e-36 of its partner's (norm ratio 1e-18)
// is numerically zero next to it (reading R29): the pair counts as converged
// and the row is replaced by an orthonormal completion at the end.
__device__ __forceinline__ bool negligible(double di, double dj) {
  return fmin(fabs(di), fabs(dj)) <= 1e-36 * fmax(fabs(di), fabs(dj));
}

// round-robin (circle method) pairing of nb players (nb even), round r, pair p
__device__ __forceinline__ void rr_pair(int nb, int r, int p, int &a, int &b) {
  const int m = nb - 1;
  if (p == 0) {
    a = m;
    b = r;
  } else {
    a = (r + p) % m;
    b = (r - p + m) % m;
  }
}

// Shared memory of one CTA. Hp (this CTA's partial Gram, read by the other
// CTAs of the cluster over DSMEM) aliases the staging ring, and A (G^H, the
// update operand) aliases H: their lifetimes do not overlap.
template <bool C>
struct __align__(16) RoundSmem {
  using E = typename Cx<C>::E;
  union {
    E stage[Cx<C>::NST][PR][Cx<C>::PITCH];
    E Hp[PR][HP];
  };
  union {
    E H[PR][HP];
    E A[PR][HP];
  };
  E G[PR][HP];
  E rph[PR / 2];
  double rc[PR / 2], rs[PR / 2], rd[PR / 2][2];
  int ri[PR / 2], rj[PR / 2], rflag[PR / 2];
  int ord[PR];
  double ev[PR];
  double red[NT / 32];
  int lowf[PR];   // row below the truncation cut (trunc_svd low-pair skipping), per pair row
  int skip;
};

template <bool C>
__device__ __forceinline__ void load_chunk(RoundSmem<C> &sm, int stg, const typename Cx<C>::E *base, int64_t ld,
                                           int64_t row_lo, int64_t row_hi, int64_t col0) {
  constexpr int CW = Cx<C>::CW;
  constexpr int PER_ROW = CW / Cx<C>::PER16;          // 16-byte copies per row segment
  constexpr int TOTAL = PR * PER_ROW;
#pragma unroll
  for (int i = threadIdx.x; i < TOTAL; i += NT) {
    const int r = i / PER_ROW, q = i % PER_ROW;
    const int64_t grow = r < SB ? row_lo + r : row_hi + (r - SB);
    const auto *src = base + grow * ld + col0 + (int64_t)q * Cx<C>::PER16;
    cp_async_zfill<16>(&sm.stage[stg][r][q * Cx<C>::PER16], src, 16);
  }
}

// Partial Gram of the 32 pair rows over chunks [c0, c1): upper 8x8 tiles
// (ti <= tj) on DMMA; warp w accumulates k-steps w, w + 8, ... of every chunk;
// warp partials are added in warp order into sm.Hp (deterministic).
template <bool C>
__device__ void gram_pass(RoundSmem<C> &sm, const typename Cx<C>::E *X, int64_t ld, int c0, int c1,
                          int64_t row_lo, int64_t row_hi) {
  constexpr int CW = Cx<C>::CW, NST = Cx<C>::NST, KW = CW / 32;   // k-steps per warp per chunk
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = c1 - c0;
  constexpr int NTILE = 10;
  double acc[NTILE][C ? 2 : 1][2];
#pragma unroll
  for (int t = 0; t < NTILE; t++)
#pragma unroll
    for (int z = 0; z < (C ? 2 : 1); z++) acc[t][z][0] = acc[t][z][1] = 0.0;

#pragma unroll
  for (int s = 0; s < NST - 1; s++) {
    if (s < nch) load_chunk<C>(sm, s, X, ld, row_lo, row_hi, (int64_t)(c0 + s) * CW);
    cp_async_commit();
  }
  for (int c = 0; c < nch; c++) {
    cp_async_wait<NST - 2>();
    __syncthreads();
    if (c + NST - 1 < nch)
      load_chunk<C>(sm, (c + NST - 1) % NST, X, ld, row_lo, row_hi, (int64_t)(c0 + c + NST - 1) * CW);
    cp_async_commit();
    const auto &st = sm.stage[c % NST];
#pragma unroll
    for (int kw = 0; kw < KW; kw++) {
      const int kc = (warp + 8 * kw) * 4 + (lane & 3);
      if constexpr (!C) {
        double f[4];
#pragma unroll
        for (int t = 0; t < 4; t++) f[t] = st[t * 8 + (lane >> 2)][kc];
        int idx = 0;
#pragma unroll
        for (int ti = 0; ti < 4; ti++)
#pragma unroll
          for (int tj = ti; tj < 4; tj++) dmma884(acc[idx++][0], f[ti], f[tj]);
      } else {
        double fr[4], fi[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
          const double2 v = st[t * 8 + (lane >> 2)][kc];
          fr[t] = v.x;
          fi[t] = v.y;
        }
        int idx = 0;
#pragma unroll
        for (int ti = 0; ti < 4; ti++)
#pragma unroll
          for (int tj = ti; tj < 4; tj++) {
            // H_ij = sum x_i conj(x_j): re = xr_i xr_j + xi_i xi_j, im = xi_i xr_j - xr_i xi_j
            dmma884(acc[idx][0], fr[ti], fr[tj]);
            dmma884(acc[idx][0], fi[ti], fi[tj]);
            dmma884(acc[idx][1], fi[ti], fr[tj]);
            dmma884(acc[idx][1], -fr[ti], fi[tj]);
            idx++;
          }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // add the warp partials in warp order (deterministic); Hp aliases the ring
  for (int w = 0; w < NT / 32; w++) {
    if (warp == w) {
      int idx = 0;
#pragma unroll
      for (int ti = 0; ti < 4; ti++)
#pragma unroll
        for (int tj = ti; tj < 4; tj++) {
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int i = ti * 8 + (lane >> 2), j = tj * 8 + 2 * (lane & 3) + e;
            if constexpr (!C) {
              sm.Hp[i][j] = w == 0 ? acc[idx][0][e] : sm.Hp[i][j] + acc[idx][0][e];
            } else {
              const double2 v = make_double2(acc[idx][0][e], acc[idx][1][e]);
              sm.Hp[i][j] = w == 0 ? v : cadd(sm.Hp[i][j], v);
            }
          }
          idx++;
        }
    }
    __syncthreads();
  }
}

// H (PR x PR Hermitian, shared) -> eigenvectors G (one Newton-Schulz step of
// re-orthonormalisation), then A = G^H with the eigenpairs of the first nreal
// rows in descending eigenvalue order (ties by index). A aliases H.
template <bool C>
__device__ void block_eig(RoundSmem<C> &sm, int nreal, double tol_in, int max_inner, int sort, double zfloor2,
                          unsigned long long *prof = nullptr) {
  using E = typename Cx<C>::E;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < PR * PR; idx += NT) sm.G[idx / PR][idx % PR] = (idx / PR == idx % PR) ? cone<E>() : czero<E>();
  __syncthreads();
  for (int sw = 0; sw < max_inner; sw++) {
    int rotated = 0;
    for (int step = 0; step < PR - 1; step++) {
      long long q0 = 0;
      if (prof && tid == 0) q0 = clock64();
      if (tid < PR / 2) {
        int a, b;
        rr_pair(PR, step, tid, a, b);
        const int i = min(a, b), j = max(a, b);
        sm.ri[tid] = i;
        sm.rj[tid] = j;
        const double hi = re(sm.H[i][i]), hj = re(sm.H[j][j]);
        const E h = sm.H[i][j];
        const double ah = cabs(h);
        // rotate only above the inner tolerance (a fraction of the outer one):
        // chasing rounding noise adds rotations with c rounded to 1, whose
        // c^2 + s^2 > 1 bias grows the row norms
        // pairs with a numerically zero row (R29) are left alone: the row is
        // completed at the end
        // rows at or below the noise floor (zfloor2, squared norm) are frozen:
        // their directions are rounding noise, completed at the end (R29)
        if (ah == 0.0 || ah <= tol_in * sqrt(fabs(hi)) * sqrt(fabs(hj)) || negligible(hi, hj) ||
            fmin(hi, hj) <= zfloor2 || (sm.lowf[i] && sm.lowf[j])) {
          sm.rflag[tid] = 0;
        } else {
          // real symmetric [[hi, |h|], [|h|, hj]] (after the phase) -> R = [[c, s], [-s, c]]
          // tau = (hj - hi) / (2|h|), t = sign(tau) / (|tau| + sqrt(1 + tau^2))
          // (scale-free: Gram entries of rows ~1e100 must not overflow)
          const double tau = (hj - hi) / (2.0 * ah);
          const double at = fabs(tau);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (at > 1e150 ? 2.0 * at : at + sqrt(fma(tau, tau, 1.0)));
          const double c = rsqrt(fma(t, t, 1.0));
          sm.rc[tid] = c;
          sm.rs[tid] = t * c;
          sm.rph[tid] = phase_of(h, ah);   // e^{-i phi}
          sm.rd[tid][0] = hi - t * ah;
          sm.rd[tid][1] = hj + t * ah;
          sm.rflag[tid] = 1;
          rotated = 1;
        }
      }
      __syncthreads();
      long long q1 = 0;
      if (prof && tid == 0) {
        q1 = clock64();
        atomicAdd(prof + 5, (unsigned long long)(q1 - q0));
      }
      {
        // H <- J^H H J on 2x2 blocks (u, v), J_u = [[c, s], [-s ph, c ph]]
        const int u = tid >> 4, v = tid & 15;
        if (u <= v && (sm.rflag[u] | sm.rflag[v])) {
          const int iu = sm.ri[u], ju = sm.rj[u], iv = sm.ri[v], jv = sm.rj[v];
          if (u == v) {
            sm.H[iu][iu] = rmul(sm.rd[u][0], cone<E>());
            sm.H[ju][ju] = rmul(sm.rd[u][1], cone<E>());
            sm.H[iu][ju] = czero<E>();
            sm.H[ju][iu] = czero<E>();
          } else {
            E b00 = sm.H[iu][iv], b01 = sm.H[iu][jv], b10 = sm.H[ju][iv], b11 = sm.H[ju][jv];
            if (sm.rflag[v]) {   // T = B J_v
              const double c = sm.rc[v], s = sm.rs[v];
              const E ph = sm.rph[v];
              const E t00 = cadd(rmul(c, b00), rmul(-s, cmul(b01, ph)));
              const E t01 = cadd(rmul(s, b00), rmul(c, cmul(b01, ph)));
              const E t10 = cadd(rmul(c, b10), rmul(-s, cmul(b11, ph)));
              const E t11 = cadd(rmul(s, b10), rmul(c, cmul(b11, ph)));
              b00 = t00; b01 = t01; b10 = t10; b11 = t11;
            }
            if (sm.rflag[u]) {   // M = J_u^H T, J_u^H = [[c, -s conj(ph)], [s, c conj(ph)]]
              const double c = sm.rc[u], s = sm.rs[u];
              const E pc = cj(sm.rph[u]);
              const E m00 = cadd(rmul(c, b00), rmul(-s, cmul(pc, b10)));
              const E m01 = cadd(rmul(c, b01), rmul(-s, cmul(pc, b11)));
              const E m10 = cadd(rmul(s, b00), rmul(c, cmul(pc, b10)));
              const E m11 = cadd(rmul(s, b01), rmul(c, cmul(pc, b11)));
              b00 = m00; b01 = m01; b10 = m10; b11 = m11;
            }
            sm.H[iu][iv] = b00; sm.H[iu][jv] = b01; sm.H[ju][iv] = b10; sm.H[ju][jv] = b11;
            sm.H[iv][iu] = cj(b00); sm.H[jv][iu] = cj(b01); sm.H[iv][ju] = cj(b10); sm.H[jv][ju] = cj(b11);
          }
        }
        // G <- G J: rows r, pairs v
        for (int it = tid; it < PR * (PR / 2); it += NT) {
          const int r = it >> 4, w = it & 15;
          if (sm.rflag[w]) {
            const int iw = sm.ri[w], jw = sm.rj[w];
            const double c = sm.rc[w], s = sm.rs[w];
            const E ph = sm.rph[w];
            const E gi = sm.G[r][iw], gj = sm.G[r][jw];
            sm.G[r][iw] = cadd(rmul(c, gi), rmul(-s, cmul(gj, ph)));
            sm.G[r][jw] = cadd(rmul(s, gi), rmul(c, cmul(gj, ph)));
          }
        }
      }
      __syncthreads();
      if (prof && tid == 0) atomicAdd(prof + 6, (unsigned long long)(clock64() - q1));
    }
    if (!__syncthreads_or(rotated)) break;
  }
  if (tid < PR) sm.ev[tid] = re(sm.H[tid][tid]);
  __syncthreads();
  // one Newton-Schulz step G <- G (3 I - G^H G) / 2 restores unitarity to
  // rounding level (the rotations' c^2 + s^2 - 1 errors otherwise accumulate
  // over the sweeps in X and Y); A (= H's storage) holds G^H G meanwhile
  for (int idx = tid; idx < PR * PR; idx += NT) {
    const int i = idx / PR, j = idx % PR;
    E acc = czero<E>();
    for (int r = 0; r < PR; r++) acc = cadd(acc, cmul(cj(sm.G[r][i]), sm.G[r][j]));
    sm.A[i][j] = acc;
  }
  __syncthreads();
  E gn[PR * PR / NT];
#pragma unroll
  for (int q = 0; q < PR * PR / NT; q++) {
    const int idx = tid + q * NT, r = idx / PR, j = idx % PR;
    E acc = czero<E>();
    for (int i = 0; i < PR; i++) acc = cadd(acc, cmul(sm.G[r][i], sm.A[i][j]));
    gn[q] = cadd(rmul(1.5, sm.G[r][j]), rmul(-0.5, acc));
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PR * PR / NT; q++) {
    const int idx = tid + q * NT;
    sm.G[idx / PR][idx % PR] = gn[q];
  }
  // descending eigenvalue order (ties by index) among the first nreal rows;
  // padding rows (global index >= n, a suffix of the pair) keep their place,
  // so they stay exact zero rows of X and unit rows of Y
  if (tid < PR) {
    if (tid < nreal && sort) {
      const double e = sm.ev[tid];
      int rank = 0;
      for (int j = 0; j < nreal; j++) {
        const double f = sm.ev[j];
        rank += (f > e) || (f == e && j < tid);
      }
      sm.ord[rank] = tid;
    } else {
      sm.ord[tid] = tid;
    }
  }
  __syncthreads();
  for (int idx = tid; idx < PR * PR; idx += NT) {
    const int k = idx / PR, j = idx % PR;
    sm.A[k][j] = cj(sm.G[j][sm.ord[k]]);
  }
  __syncthreads();
}

// rows <- A rows over chunks [c0, c1) of one matrix (in place), A = G^H
// the first NST - 1 chunk loads of an update pass (issued early by the caller
// so they overlap the eigensolver)
template <bool C>
__device__ __forceinline__ void update_prologue(RoundSmem<C> &sm, const typename Cx<C>::E *X, int64_t ld, int c0,
                                                int c1, int64_t row_lo, int64_t row_hi) {
#pragma unroll
  for (int s = 0; s < Cx<C>::NST - 1; s++) {
    if (s < c1 - c0) load_chunk<C>(sm, s, X, ld, row_lo, row_hi, (int64_t)(c0 + s) * Cx<C>::CW);
    cp_async_commit();
  }
}

template <bool C>
__device__ void update_pass(RoundSmem<C> &sm, typename Cx<C>::E *X, int64_t ld, int c0, int c1, int64_t row_lo,
                            int64_t row_hi, bool prologue_done = false) {
  constexpr int CW = Cx<C>::CW, NST = Cx<C>::NST, TW = CW / 16;   // column tiles per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = warp >> 1, tj0 = TW * (warp & 1);
  const int nch = c1 - c0;
  // A fragments of row tile ti for the 8 k-steps (kept in registers)
  double ar[8], ai[8];
#pragma unroll
  for (int kk = 0; kk < 8; kk++) {
    const auto v = sm.A[ti * 8 + (lane >> 2)][kk * 4 + (lane & 3)];
    if constexpr (!C) {
      ar[kk] = v;
      ai[kk] = 0.0;
    } else {
      ar[kk] = v.x;
      ai[kk] = v.y;
    }
  }
  const int orow = ti * 8 + (lane >> 2);
  const int64_t grow = orow < SB ? row_lo + orow : row_hi + (orow - SB);
if (!prologue_done) update_prologue<C>(sm, X, ld, c0, c1, row_lo, row_hi);
  for (int c = 0; c < nch; c++) {
    cp_async_wait<NST - 2>();
    __syncthreads();
    if (c + NST - 1 < nch)
      load_chunk<C>(sm, (c + NST - 1) % NST, X, ld, row_lo, row_hi, (int64_t)(c0 + c + NST - 1) * CW);
    cp_async_commit();
    const auto &st = sm.stage[c % NST];
    double acc[TW][C ? 2 : 1][2];
#pragma unroll
    for (int t = 0; t < TW; t++)
#pragma unroll
      for (int z = 0; z < (C ? 2 : 1); z++) acc[t][z][0] = acc[t][z][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; kk++) {
#pragma unroll
      for (int t = 0; t < TW; t++) {
        const auto b = st[kk * 4 + (lane & 3)][(tj0 + t) * 8 + (lane >> 2)];
        if constexpr (!C) {
          dmma884(acc[t][0], ar[kk], b);
        } else {
          dmma884(acc[t][0], ar[kk], b.x);    // re += ar br - ai bi
          dmma884(acc[t][0], -ai[kk], b.y);
          dmma884(acc[t][1], ar[kk], b.y);    // im += ar bi + ai br
          dmma884(acc[t][1], ai[kk], b.x);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < TW; t++) {
      const int64_t col = (int64_t)(c0 + c) * CW + (tj0 + t) * 8 + 2 * (lane & 3);
      auto *dst = X + grow * ld + col;
      if constexpr (!C) {
        *reinterpret_cast<double2 *>(dst) = make_double2(acc[t][0][0], acc[t][0][1]);
      } else {
        dst[0] = make_double2(acc[t][0][0], acc[t][1][0]);
        dst[1] = make_double2(acc[t][0][1], acc[t][1][1]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// One round: cluster q (CL CTAs) handles block pair q; CTA rank r of the
// cluster owns the r-th contiguous slice of the column chunks of X and Y.
template <bool C>
__global__ void __launch_bounds__(NT, 2) svd_round_kernel(typename Cx<C>::E *X, int64_t ldx, typename Cx<C>::E *Y,
                                                          int64_t ldy, int nb, int64_t n, int round, double tol,
                                                          double tol_in, int max_inner, double zfloor2,
                                                          const int *low, unsigned long long *offmax,
                                                          unsigned long long *prof) {
  using E = typename Cx<C>::E;
  constexpr int CW = Cx<C>::CW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RoundSmem<C> &sm = *reinterpret_cast<RoundSmem<C> *>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  int a, b;
  rr_pair(nb, round, blockIdx.x / CL, a, b);
  const int64_t row_lo = (int64_t)min(a, b) * SB, row_hi = (int64_t)max(a, b) * SB;
  const int nchx = (int)(ldx / CW), nchy = (int)(ldy / CW);
  const int x0 = (int)((int64_t)nchx * rank / CL), x1 = (int)((int64_t)nchx * (rank + 1) / CL);
  const int y0 = (int)((int64_t)nchy * rank / CL), y1 = (int)((int64_t)nchy * (rank + 1) / CL);

  long long tp0 = 0;
  if (prof && threadIdx.x == 0) tp0 = clock64();
  gram_pass<C>(sm, X, ldx, x0, x1, row_lo, row_hi);
  if (prof && threadIdx.x == 0) atomicAdd(prof + 0, (unsigned long long)(clock64() - tp0));
  // H = sum of the cluster's partials in rank order (identical in every CTA)
  cluster.sync();
  for (int idx = threadIdx.x; idx < PR * PR; idx += NT) {
    const int i = idx / PR, j = idx % PR;
    if (i <= j) {
      E acc = czero<E>();
      for (int q = 0; q < CL; q++) acc = cadd(acc, cluster.map_shared_rank(&sm.Hp[0][0], q)[i * HP + j]);
      sm.H[i][j] = acc;
    }
  }
  cluster.sync();   // remote reads of Hp done before the ring is reused
  // Hermitian completion from the upper triangle; real diagonal
  for (int idx = threadIdx.x; idx < PR * PR; idx += NT) {
    const int i = idx / PR, j = idx % PR;
    if (i > j) sm.H[i][j] = cj(sm.H[j][i]);
    if constexpr (C) {
      if (i == j) sm.H[i][i].y = 0.0;
    }
  }
  __syncthreads();

  // rows below the truncation cut (both rows of a pair low: the pair only
  // mixes discarded rows and is skipped, trunc_svd with chi_max < n)
  for (int i = threadIdx.x; i < PR; i += NT) {
    const int64_t r = i < SB ? row_lo + i : row_hi + (i - SB);
    sm.lowf[i] = (low && r < n) ? low[r] : 0;
  }
  __syncthreads();
  // convergence test: max relative off-diagonal |H_ij| / sqrt(H_ii H_jj)
  double off = 0.0;
  for (int idx = threadIdx.x; idx < PR * PR; idx += NT) {
    const int i = idx / PR, j = idx % PR;
    if (i < j) {
      const double di = re(sm.H[i][i]), dj = re(sm.H[j][j]);
      if (di > zfloor2 && dj > zfloor2 && !negligible(di, dj) && !(sm.lowf[i] && sm.lowf[j]))
        off = fmax(off, cabs(sm.H[i][j]) / sqrt(di * dj));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
  if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = off;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < NT / 32; w++) m = fmax(m, sm.red[w]);
    if (rank == 0) atomicMax(offmax, (unsigned long long)__double_as_longlong(m));   // >= 0: integer order
    sm.skip = !(m > tol);
  }
  __syncthreads();
  if (sm.skip) return;   // same decision in every CTA of the cluster (identical H)

  const int64_t lo_real = n - row_lo < 0 ? 0 : (n - row_lo > SB ? SB : n - row_lo);
  const int64_t hi_real = n - row_hi < 0 ? 0 : (n - row_hi > SB ? SB : n - row_hi);
  // real rows form a prefix of the pair's row list (padding rows are the top indices)
  // the staging ring is free now (Hp was consumed): start streaming X for
  // the update while the eigensolver runs
  update_prologue<C>(sm, X, ldx, x0, x1, row_lo, row_hi);
  long long tp1 = 0;
  if (prof && threadIdx.x == 0) tp1 = clock64();
  block_eig<C>(sm, lo_real < SB ? (int)lo_real : SB + (int)hi_real, tol_in, max_inner & 0xff, (max_inner >> 8) & 1,
               zfloor2, prof);
  long long tp2 = 0;
  if (prof && threadIdx.x == 0) {
    tp2 = clock64();
    atomicAdd(prof + 1, (unsigned long long)(tp2 - tp1));
  }
  update_pass<C>(sm, X, ldx, x0, x1, row_lo, row_hi, true);
  long long tp3 = 0;
  if (prof && threadIdx.x == 0) {
    tp3 = clock64();
    atomicAdd(prof + 2, (unsigned long long)(tp3 - tp2));
  }
  update_pass<C>(sm, Y, ldy, y0, y1, row_lo, row_hi);
  if (prof && threadIdx.x == 0) {
    atomicAdd(prof + 3, (unsigned long long)(clock64() - tp3));
    atomicAdd(prof + 4, 1ull);
  }
}

// X[r][c] = A'[r][c] (wide) or conj(A'[c][r]) (tall), zero padded; 32x32 tiles
template <bool C>
__global__ void __launch_bounds__(256) svd_load_kernel(const typename Cx<C>::E *A, int64_t I, int64_t J, int tall,
                                                        typename Cx<C>::E *X, int64_t ldx) {
  using E = typename Cx<C>::E;
  __shared__ E tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (!tall) {
    for (int y = ty; y < 32; y += 8) {
      const int64_t r = r0 + y, c = c0 + tx;
      X[r * ldx + c] = (r < I && c < J) ? A[r * J + c] : czero<E>();
    }
  } else {
    // X[r][c] = conj(A[c][r]), r < J, c < I: read A rows c0.. (coalesced along r)
    for (int y = ty; y < 32; y += 8) {
      const int64_t ar = c0 + y, ac = r0 + tx;
      tile[y][tx] = (ar < I && ac < J) ? cj(A[ar * J + ac]) : czero<E>();
    }
    __syncthreads();
    for (int y = ty; y < 32; y += 8) X[(r0 + y) * ldx + c0 + tx] = tile[tx][y];
  }
}

template <bool C>
__global__ void svd_eye_kernel(typename Cx<C>::E *Y, int64_t n, int64_t ldy) {
  using E = typename Cx<C>::E;
  const int64_t total = n * ldy;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    Y[i] = (i / ldy == i % ldy) ? cone<E>() : czero<E>();
}

// s[r] = sqrt(sum_c |X[r][c]|^2): one warp per row, fixed order
template <bool C>
__global__ void __launch_bounds__(256) svd_norms_kernel(const typename Cx<C>::E *X, int64_t ldx, int64_t ncols,
                                                         int64_t nrows, double *s) {
  const int64_t r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= nrows) return;
  double acc = 0.0;
  for (int64_t c = lane; c < ncols; c += 32) {
    const auto v = X[r * ldx + c];
    if constexpr (!C) {
      acc = fma(v, v, acc);
    } else {
      acc = fma(v.x, v.x, acc);
      acc = fma(v.y, v.y, acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) s[r] = sqrt(acc);
}

// dst[k][c] = f(src[perm[k]][c]), f = optional conj, optional division by s[perm[k]]
template <bool C>
__global__ void svd_gather_rows_kernel(typename Cx<C>::E *dst, int64_t ld_dst, const typename Cx<C>::E *src,
                                       int64_t ld_src, const int *perm, const double *s, int64_t nk, int64_t ncols,
                                       int conj) {
  using E = typename Cx<C>::E;
  const int64_t k = blockIdx.y;
  if (k >= nk) return;
  const int64_t r = perm[k];
  const double sv = s ? s[r] : 1.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols; c += (int64_t)gridDim.x * blockDim.x) {
    E v = src[r * ld_src + c];
    if (conj) v = cj(v);
    if (s) {   // zero rows stay zero here (completed separately)
      if (!(sv > 0.0)) v = czero<E>();
      else if constexpr (!C) v = v / sv;
      else v = make_double2(v.x / sv, v.y / sv);
    }
    dst[k * ld_dst + c] = v;
  }
}

// dst[r][k] = f(src[perm[k]][r]) for r < nr, k < nk (dst row-major nr x nk)
template <bool C>
__global__ void __launch_bounds__(256) svd_gather_t_kernel(typename Cx<C>::E *dst, const typename Cx<C>::E *src,
                                                            int64_t ld_src, const int *perm, const double *s,
                                                            int64_t nk, int64_t nr, int conj) {
  using E = typename Cx<C>::E;
  __shared__ E tile[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int y = ty; y < 32; y += 8) {
    const int64_t k = k0 + y, r = r0 + tx;
    E v = czero<E>();
    if (k < nk && r < nr) {
      const int64_t row = perm[k];
      v = src[row * ld_src + r];
      if (conj) v = cj(v);
      if (s) {
        const double sv = s[row];
        if (sv > 0.0) {
          if constexpr (!C) v = v / sv;
          else v = make_double2(v.x / sv, v.y / sv);
        } else {
          v = czero<E>();
        }
      }
    }
    tile[y][tx] = v;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = r0 + y, k = k0 + tx;
    if (r < nr && k < nk) dst[r * nk + k] = tile[tx][y];
  }
}

// s_out[k] = s[perm[k]]
__global__ void svd_gather_s_kernel(double *s_out, const double *s, const int *perm, int64_t nk) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nk; k += (int64_t)gridDim.x * blockDim.x)
    s_out[k] = s[perm[k]];
}

// Numerically zero selected rows (s <= 1e-18 s_0, R29: the factor is undetermined there) become
// unit vectors orthogonal to every other selected row: for candidates e_j,
// j = 0, 1, ..., two Gram-Schmidt passes against the normalized selected rows
// (x_r / snorm[r], snorm[r] > 0), accepted when the residual norm > 1/(2 sqrt L).
// One CTA, sequential over zero rows; only degenerate inputs get here.
template <bool C>
__device__ double cta_sum(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
  return t;
}

template <bool C>
__global__ void __launch_bounds__(1024) svd_complete_kernel(typename Cx<C>::E *X, int64_t ldx, int64_t L,
                                                             const int *sel, int64_t nsel, double *snorm,
                                                             const int *zl, int nz) {
  using E = typename Cx<C>::E;
  __shared__ double red[32];
  for (int zi = threadIdx.x; zi < nz; zi += blockDim.x) snorm[zl[zi]] = 0.0;   // not part of the basis
  __syncthreads();
  for (int zi = 0; zi < nz; zi++) {
    const int64_t z = zl[zi];
    E *v = X + z * ldx;
    // candidates e_0, e_1, ... for every zero row (those already taken are in
    // the span of the completed rows and fail the residual test)
    for (int64_t j = 0; j < L; j++) {
      for (int64_t c = threadIdx.x; c < L; c += blockDim.x) v[c] = c == j ? cone<E>() : czero<E>();
      __syncthreads();
      for (int pass = 0; pass < 2; pass++) {
        for (int64_t k = 0; k < nsel; k++) {
          const int64_t r = sel[k];
          const double sn = snorm[r];
          if (r == z || !(sn > 0.0)) continue;
          const E *x = X + r * ldx;
          double dr = 0.0, di = 0.0;   // <x_r|v> (x_r conjugated)
          for (int64_t c = threadIdx.x; c < L; c += blockDim.x) {
            if constexpr (!C) {
              dr = fma(x[c], v[c], dr);
            } else {
              dr = fma(x[c].x, v[c].x, fma(x[c].y, v[c].y, dr));
              di = fma(x[c].x, v[c].y, fma(-x[c].y, v[c].x, di));
            }
          }
          dr = cta_sum<C>(dr, red) / (sn * sn);
          if constexpr (C) di = cta_sum<C>(di, red) / (sn * sn);
          for (int64_t c = threadIdx.x; c < L; c += blockDim.x) {
            if constexpr (!C) {
              v[c] -= dr * x[c];
            } else {
              v[c].x -= dr * x[c].x - di * x[c].y;
              v[c].y -= dr * x[c].y + di * x[c].x;
            }
          }
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int64_t c = threadIdx.x; c < L; c += blockDim.x) {
        if constexpr (!C) nn = fma(v[c], v[c], nn);
        else nn = fma(v[c].x, v[c].x, fma(v[c].y, v[c].y, nn));
      }
      const double nrm = sqrt(cta_sum<C>(nn, red));
      // some e_j has a residual >= 1/sqrt(L) whenever the complement is non-empty
      if (nrm > 0.5 / sqrt((double)L)) {
        for (int64_t c = threadIdx.x; c < L; c += blockDim.x) v[c] = rmul(1.0 / nrm, v[c]);
        __syncthreads();
        if (threadIdx.x == 0) snorm[z] = 1.0;
        __syncthreads();
        break;
      }
    }
  }
}

template <bool C>
size_t round_smem() {
  return sizeof(RoundSmem<C>);
}

}  // namespace

size_t svd_round_smem_bytes(bool cplx) { return cplx ? round_smem<true>() : round_smem<false>(); }

cudaError_t launch_svd_load(const SvdProblem &p, const void *A, int64_t I, int64_t J, cudaStream_t s,
                            int64_t *launches) {
  dim3 grid((unsigned)(p.ldx / 32), (unsigned)(p.npad / 32));
  if (p.cplx)
    svd_load_kernel<true><<<grid, 256, 0, s>>>(static_cast<const double2 *>(A), I, J, p.tall,
                                               static_cast<double2 *>(p.X), p.ldx);
  else
    svd_load_kernel<false><<<grid, 256, 0, s>>>(static_cast<const double *>(A), I, J, p.tall,
                                                static_cast<double *>(p.X), p.ldx);
  (*launches)++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int blocks = 4 * 148;
  if (p.cplx)
    svd_eye_kernel<true><<<blocks, 256, 0, s>>>(static_cast<double2 *>(p.Y), p.npad, p.ldy);
  else
    svd_eye_kernel<false><<<blocks, 256, 0, s>>>(static_cast<double *>(p.Y), p.npad, p.ldy);
  (*launches)++;
  return cudaGetLastError();
}

cudaError_t launch_svd_round(const SvdProblem &p, int round, double tol, double tol_in, int max_inner,
                             cudaStream_t s, int64_t *launches) {
  const int nb = (int)(p.npad / SB);
  const int pairs = nb / 2;
  // CTAs per block pair: fill ~2 CTAs per SM on the 148 SMs (portable cluster <= 8)
  int cl = 1;
  while (cl < 8 && pairs * cl * 2 <= 2 * 148) cl *= 2;
  const size_t smem = svd_round_smem_bytes(p.cplx);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(pairs * cl));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (p.cplx) {
    auto k = svd_round_kernel<true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaLaunchKernelEx(&cfg, k, static_cast<double2 *>(p.X), p.ldx, static_cast<double2 *>(p.Y), p.ldy, nb,
                           p.n, round, tol, tol_in, max_inner, p.zfloor2, p.low, p.offmax, p.prof);
  } else {
    auto k = svd_round_kernel<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaLaunchKernelEx(&cfg, k, static_cast<double *>(p.X), p.ldx, static_cast<double *>(p.Y), p.ldy, nb, p.n,
                           round, tol, tol_in, max_inner, p.zfloor2, p.low, p.offmax, p.prof);
  }
  (*launches)++;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_svd_norms(const SvdProblem &p, cudaStream_t s, int64_t *launches) {
  const unsigned grid = (unsigned)((p.npad + 7) / 8);
  if (p.cplx)
    svd_norms_kernel<true><<<grid, 256, 0, s>>>(static_cast<const double2 *>(p.X), p.ldx, p.L, p.npad, p.s);
  else
    svd_norms_kernel<false><<<grid, 256, 0, s>>>(static_cast<const double *>(p.X), p.ldx, p.L, p.npad, p.s);
  (*launches)++;
  return cudaGetLastError();
}

cudaError_t launch_svd_gather_rows(bool cplx, void *dst, int64_t ld_dst, const void *src, int64_t ld_src,
                                   const int *perm, const double *s, int64_t nk, int64_t ncols, int conj,
                                   cudaStream_t st, int64_t *launches) {
  if (nk == 0 || ncols == 0) return cudaSuccess;
  dim3 grid((unsigned)std::min<int64_t>((ncols + 255) / 256, 64), (unsigned)nk);
  if (cplx)
    svd_gather_rows_kernel<true><<<grid, 256, 0, st>>>(static_cast<double2 *>(dst), ld_dst,
                                                       static_cast<const double2 *>(src), ld_src, perm, s, nk, ncols,
                                                       conj);
  else
    svd_gather_rows_kernel<false><<<grid, 256, 0, st>>>(static_cast<double *>(dst), ld_dst,
                                                        static_cast<const double *>(src), ld_src, perm, s, nk, ncols,
                                                        conj);
  (*launches)++;
  return cudaGetLastError();
}

cudaError_t launch_svd_gather_t(bool cplx, void *dst, const void *src, int64_t ld_src, const int *perm,
                                const double *s, int64_t nk, int64_t nr, int conj, cudaStream_t st,
                                int64_t *launches) {
  if (nk == 0 || nr == 0) return cudaSuccess;
  dim3 grid((unsigned)((nk + 31) / 32), (unsigned)((nr + 31) / 32));
  if (cplx)
    svd_gather_t_kernel<true><<<grid, 256, 0, st>>>(static_cast<double2 *>(dst), static_cast<const double2 *>(src),
                                                    ld_src, perm, s, nk, nr, conj);
  else
    svd_gather_t_kernel<false><<<grid, 256, 0, st>>>(static_cast<double *>(dst), static_cast<const double *>(src),
                                                     ld_src, perm, s, nk, nr, conj);
  (*launches)++;
  return cudaGetLastError();
}

cudaError_t launch_svd_gather_s(double *s_out, const double *s, const int *perm, int64_t nk, cudaStream_t st,
                                int64_t *launches) {
  if (nk == 0) return cudaSuccess;
  svd_gather_s_kernel<<<(unsigned)std::min<int64_t>((nk + 255) / 256, 1024), 256, 0, st>>>(s_out, s, perm, nk);
  (*launches)++;
  return cudaGetLastError();
}

cudaError_t launch_svd_complete(const SvdProblem &p, const int *sel, int64_t nsel, double *snorm, const int *zl,
                                int nz, cudaStream_t st, int64_t *launches) {
  if (nz == 0) return cudaSuccess;
  if (p.cplx)
    svd_complete_kernel<true><<<1, 1024, 0, st>>>(static_cast<double2 *>(p.X), p.ldx, p.L, sel, nsel, snorm, zl, nz);
  else
    svd_complete_kernel<false><<<1, 1024, 0, st>>>(static_cast<double *>(p.X), p.ldx, p.L, sel, nsel, snorm, zl, nz);
  (*launches)++;
  return cudaGetLastError();
}

}  // namespace tci
