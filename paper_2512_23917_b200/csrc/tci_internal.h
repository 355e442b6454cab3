// tci_internal.h -- internal declarations shared by the C ABI layer, the
// planner and the CUDA kernels of libtci_b200. Not installed; not part of
// the ABI (include/tci_b200.h is).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/tci_b200.h"

namespace tci {

// Host-side launch-attribute caches (launch_cache.cpp): the dynamic shared
// memory opt-in of a kernel (set only when `bytes` exceeds what was set for
// that kernel on this device), blocks per SM from the occupancy calculator,
// and the SM count -- answered from tables after the first call.
cudaError_t ensure_smem_attr(const void *fn, size_t bytes);
int occupancy_per_sm(const void *fn, int threads, size_t smem);
int device_sms();

constexpr int kMaxOrder = TCI_MAX_ORDER;

inline size_t dtype_size(tci_dtype_t t) {
  switch (t) {
    case TCI_R32: return 4;
    case TCI_R64: return 8;
    case TCI_C64: return 8;
    case TCI_C128: return 16;
  }
  return 0;
}
inline bool dtype_is_complex(tci_dtype_t t) { return t == TCI_C64 || t == TCI_C128; }

// ---------------------------------------------------------------------------
// GEMM over fused legs: C[m,n] = sum_k A(m,k) B(k,n).
// Offsets are in ELEMENTS of the dtype (a complex element = (re,im) pair).
//   A(m,k) at A + m*a_sm + k*a_sk, exactly one of a_sm/a_sk is 1 (or both
//   when the extent is 1); same for B(k,n) and C(m,n) (c_sn == 1 required:
//   the planner swaps operands to reach an N-contiguous C).
// ---------------------------------------------------------------------------
struct GemmProblem {
  tci_dtype_t dtype;
  int64_t M, N, K;
  const void *A; int64_t a_sm, a_sk;
  const void *B; int64_t b_sk, b_sn;
  void *C; int64_t c_sm;        // c_sn == 1
  // complex128 algorithm (kZ3M / kZ4M on DMMA, kZOzaki on INT8 tcgen05) and,
  // for kZOzaki, its scratch (ozaki_workspace_bytes)
  int zalgo = 0;
  void *oz_ws = nullptr;
  size_t oz_ws_bytes = 0;
  struct OzProf *oz_prof = nullptr;   // optional: event timing of the INT8 GEMMs
  // Ozaki accuracy guard (R26): when oz_tol > 0 the estimated
  // relative Frobenius truncation error of the product is compared on the
  // device with oz_tol and, if larger, the GEMM is recomputed on DMMA (a
  // DMMA launch gated by a device flag); oz_guard (device, context-owned)
  // accumulates statistics. oz_balance = 0 disables the K-balancing.
  double oz_tol = 0.0;
  struct OzGuard *oz_guard = nullptr;
  int oz_balance = 1;
  // complex Ozaki GEMMs: Gaussian moduli, two planes per modulus (1, R33) or
  // the 3M split, three planes per modulus (0)
  int oz_gauss = 1;
  // DMMA kernels: when set, every CTA returns at once unless *run_if != 0
  const int *run_if = nullptr;
  // deterministic split-K (few output tiles, long K): split z of `splitk`
  // sums k in [z*k_chunk, min(K,(z+1)*k_chunk)) into partial + z*M*N (double
  // or double2 elements, row-major [M][N]); a reduce kernel then adds the
  // splits in ascending z into C. k_chunk is a multiple of 16.
  int splitk = 1;
  int64_t k_chunk = 0;
  void *partial = nullptr;
  // mode 1 = TEBD theta with the gate in the epilogue (launch_tebd_fused)
  int mode = 0;
  // gamma-order scatter epilogue: when c_row is set, C(m, n)
  // is stored at c_row[m] + c_col[n] (device tables, elements) instead of
  // m * c_sm + n; split-K partials stay dense and the reduction scatters
  const int64_t *c_row = nullptr, *c_col = nullptr;
  // optional: called (host side, at enqueue time) after the kernels that
  // finish output rows [m0, m0 + mc) have been enqueued on the stream -- the
  // Ozaki path calls it per row chunk (at most max_chunk_rows rows when > 0),
  // so a caller can stream finished rows out while later rows compute
  void (*rows_done)(void *user, int64_t m0, int64_t mc) = nullptr;
  // optional: called (host side) before the kernels that READ rows [m0,
  // m0 + mc) of A are enqueued (the caller may make the stream wait for them
  // to arrive); with it the Ozaki path also takes A's row exponents per chunk
  void (*rows_needed)(void *user, int64_t m0, int64_t mc) = nullptr;
  void *rows_user = nullptr;
  int64_t max_chunk_rows = 0;
  // peer-memory all-gather fused into the epilogue (Ozaki CRT only): every
  // stored C element is also stored at the same offset from peer_C[p]
  // (another rank's buffer, mapped over NVLink); c_row must be null
  int npeer = 0;
  void *peer_C[7] = {};
  int64_t te_chi_a = 0, te_chi_c = 0;     // extents of a and c
  int64_t te_a_a = 0, te_a_s = 0;         // A strides of a and s (b stride == 1)
  int64_t te_b_t = 0;                     // B stride of t (c stride == 1, b stride = b_sk)
  const double *te_U = nullptr;           // gate U[p,q,s,t], device
  int64_t te_u[4] = {0, 0, 0, 0};         // strides of p, q, s, t in U
  double *te_T = nullptr;                 // theta
  int64_t te_t[4] = {0, 0, 0, 0};         // strides of a, p, q, c in theta
};

enum { kZ3M = 0, kZ4M = 1, kZOzaki = 2 };
// event pairs around each INT8 tensor-core GEMM of an Ozaki GEMM, with its
// executed int8 ops (2 per MAC over the padded batch); filled by ozaki.cu
struct OzProf {
  int n;
  cudaEvent_t a[64], b[64];
  double ops[64];
};
// Device-resident statistics of the Ozaki accuracy guard (one per context,
// written by one thread of the guard kernel, stream-ordered)
struct OzGuard {
  unsigned long long gemms;       // Ozaki GEMMs checked
  unsigned long long fallbacks;   // of which recomputed on DMMA
  unsigned long long balanced;    // of which ran with a non-trivial K-balancing
  double last_est;                // estimated relative Frobenius error of the last one
  double max_est;                 // maximum over all since the last reset
};
constexpr double kOzakiDefaultTol = 1e-13;
// the guard's tolerance for float32 / complex64 Ozaki GEMMs (R34: 100x under
// the 1e-5 fp32 bar)
constexpr double kOzakiF32Tol = 1e-7;
// The DMMA path for p (complex 3M / float64), every CTA gated by *run_if
// (gemm_dmma.cu): the Ozaki guard's recomputation
cudaError_t launch_gemm_dmma_if(const GemmProblem &p, const int *run_if, cudaStream_t s, int64_t *launches);
// Scratch of the Ozaki-II INT8 complex GEMM (ozaki.cu) for an M x N x K product.
size_t ozaki_workspace_bytes(int64_t M, int64_t N, int64_t K);
// float64 on the same scheme: one residue plane per modulus (ozaki.cu)
cudaError_t launch_ozaki_dgemm(const GemmProblem &g, void *ws, size_t ws_bytes, cudaStream_t s,
                               int64_t *launches);
cudaError_t launch_ozaki_zgemm(const GemmProblem &g, void *ws, size_t ws_bytes, cudaStream_t s,
                               int64_t *launches);
// Ozaki pays ~10 passes over the operands: use it only for big products.
// K <= 131072 keeps every int32 residue dot product exact (K * 127^2 < 2^31).
constexpr int64_t kOzakiMaxK = 131072;
// Beyond the size gate, a cost model (seconds at measured B200 rates): the
// INT8 GEMMs, the residue planes of both operands, and the byte planes the
// GEMM writes + the CRT reads + the output, against the DMMA (float64 /
// complex128) or FP64-core (float32 / complex64) GEMM. Short K loses: the
// CRT's M N (2 planes + out) bytes then outweigh 2 M N K flops (sweep
// instances with K = 64..80 ran 3-9x slower on the INT8 path).
inline bool ozaki_worthwhile(int64_t M, int64_t N, int64_t K, tci_dtype_t dt = TCI_C128) {
  if (!((double)M * (double)N * (double)K >= 4.0e9 && M >= 256 && N >= 256 && K >= 64 && K <= kOzakiMaxK))
    return false;
  const bool cplx = dt == TCI_C128 || dt == TCI_C64, f32 = dt == TCI_R32 || dt == TCI_C64;
  const double planes = cplx ? (f32 ? 20.0 : 30.0) : (f32 ? 9.0 : 14.0);
  const double es = (cplx ? 16.0 : 8.0) / (f32 ? 2.0 : 1.0);
  const double mnk = (double)M * (double)N * (double)K, mn = (double)M * (double)N;
  const double t_oz = planes * 2.0 * mnk / 2.8e15 + (double)(M + N) * (double)K * (es + planes) / 5e12 +
                      mn * (2.0 * planes + es) / 5e12;
  const double t_alt = (cplx ? 8.0 : 2.0) * mnk / (f32 ? (cplx ? 25e12 : 30e12) : (cplx ? 45e12 : 35e12));
  return t_oz < 0.8 * t_alt;
}
// The residue products of one Ozaki GEMM in one launch (i8gemm.cu, tcgen05
// kind::i8): D[b] = (A[b] B[b]^T) mod m_(b / per_mod) over L planes,
// A [L][M][Kp], B [L][N][Kp] int8 K-major, D [L][M][N] uint8; moduli[nmod]
// (odd, 64 < m < 256, L <= per_mod * nmod); counter: one device int of
// scratch (dynamic tile schedule)
cudaError_t launch_i8gemm(const int8_t *A, const int8_t *B, uint8_t *D, int64_t M, int64_t N, int64_t Kp, int L,
                          int per_mod, const int *moduli, int nmod, int *counter, cudaStream_t s,
                          int64_t *launches);
// The Ozaki CRT on the INT8 tensor cores (crt_mma.cu): the residue planes
// D [planes][Mc][Np] (complex: planes = 2n <= 32; real: n) times the base-256
// digits Bd[k][j] of the CRT weights (columns 0..15 Re / the real value,
// 16..31 Im, zero for real outputs), then the
// exact digit -> double reconstruction and the 2^(-2t + E_m + E_n) scaling
// into C (complex128, or complex64 when f32_out); guard row sums in
// rowsq[m * slots_per_row + ...] (crt_mma_slots_per_row(Np) slots per row)
struct CrtMmaArgs {
  const uint8_t *D;
  int64_t Mc, N, Np, m0;
  int planes, nd;              // residue planes, base-256 digits of M
  uint8_t Bd[32][32];
  double Mch[4];               // 32-bit chunks of M
  double Minv;                 // ~2^(32 (NC - 2)) / M (NC: 32-bit chunks of the epilogue)
  const int *EA, *EB;
  int t;
  void *C;
  int64_t c_sm;
  int npeer;
  void *peer[7];
  double *rowsq;
  int64_t slots_per_row;
  const int *eb_max;
};
cudaError_t launch_crt_mma(const CrtMmaArgs &a, bool f32_out, bool real, cudaStream_t s);
int64_t crt_mma_slots_per_row(int64_t Np);
cudaError_t crt_mma_preload();   // load every instance now (see ozaki_preload)

// moduli count and integer bit budget chosen for a contraction length K;
// kind 0 = float64, 1 = complex 3M, 2 = complex Gaussian (roots j_l with
// j_l^2 = -1 mod m_l; null for the other kinds)
void ozaki_params(int64_t K, int kind, int *nmod, int *t, const int **moduli, const int **roots, int tmin = 46);
constexpr int kOzakiTminF32 = 24;   // float32 / complex64 sources (R34; ozaki.cu kOzTminF32)


// Output tile of the GEMM kernel used for `dtype` (for the planner's split-K choice).
void gemm_tile(tci_dtype_t dtype, int *bm, int *bn);

// HBM-bound GEMM corners (gemm_thin.cu): min(M, N) <= 32 (16 complex; any K, honours the
// split-K fields) or K <= 16 (no split-K). launch_gemm dispatches to it.
bool gemm_thin_applies(const GemmProblem &p);
cudaError_t launch_gemm_thin(const GemmProblem &p, cudaStream_t s, int64_t *launches);

// Launches the DMMA (f64/c128) or FFMA (f32/c64) GEMM. Returns cudaSuccess or
// the launch error. `launches` is incremented per kernel launched.
cudaError_t launch_gemm(const GemmProblem &p, cudaStream_t s, int64_t *launches);

// TEBD theta with the gate applied in the GEMM epilogue.
// C = A.B with A rows (a,s) = m, B cols (t,c) = n; theta[a,p,q,c] written at
// a*t_a + p*t_p + q*t_q + c*t_c. d = 2 only. Real f64 only.
struct TebdProblem {
  int64_t chi_a, chi_b, chi_c, d;
  const double *A; int64_t a_a, a_s, a_b;   // strides (elements)
  const double *B; int64_t b_b, b_t, b_c;
  const double *U; int64_t u_p, u_q, u_s, u_t;   // gate (device) and its strides
  double *T; int64_t t_a, t_p, t_q, t_c;
};
cudaError_t launch_tebd_fused(const TebdProblem &p, cudaStream_t s, int64_t *launches);
bool tebd_fused_supported(const TebdProblem &p);
// the same with TMA-loaded operand tiles (tebd_tma.cu; config 3's
// "TMA-fused permutes"): natural and physical-first layouts
cudaError_t launch_tebd_tma(const TebdProblem &p, cudaStream_t s, int64_t *launches);
bool tebd_tma_supported(const TebdProblem &p);

// ---------------------------------------------------------------------------
// Permute: out[c_out] = in[c_in], c_in[perm[k]] = c_out[k].
// Shapes are already leg-fused by the caller.
// ---------------------------------------------------------------------------
struct PermuteProblem {
  int n;                       // order after fusion (0..16)
  int64_t shape_out[kMaxOrder];
  int64_t in_stride_for_out[kMaxOrder];   // stride in `in` of out bond k
  size_t esize;                // element bytes (4, 8, 16)
  const void *in;
  void *out;
  int64_t total;
};
cudaError_t launch_permute(const PermuteProblem &p, cudaStream_t s, int64_t *launches);

// ---------------------------------------------------------------------------
// Skinny small-K contraction:
//   out[b0,b1,b2, n] = sum_k in[b0,b1,b2, k] * W(k, n)
// with arbitrary per-leg strides: the fused k / n leg groups are described by
// offset tables passed BY VALUE in the kernel parameters (no device staging,
// no workspace): in(k) at in_koff[k], out(n) at out_noff[n], W(k,n) at
// w_koff[k] + w_noff[n]. Batch leg b2 is the coalesced leg. f64 / c128.
// ---------------------------------------------------------------------------
constexpr int kSkinnyMaxK = 128;
constexpr int kSkinnyMaxN = 128;
struct SkinnyProblem {
  tci_dtype_t dtype;
  int64_t nb[3];               // batch extents
  int64_t in_sb[3], out_sb[3]; // batch strides (elements)
  int K, N;
  int k_lo, n_lo;              // coalescing hints: trailing k / n runs interleaved with b2
  const void *in;
  const void *W;
  void *out;
  int64_t in_koff[kSkinnyMaxK];
  int64_t out_noff[kSkinnyMaxN];
  int32_t w_koff[kSkinnyMaxK];
  int32_t w_noff[kSkinnyMaxN];
};
cudaError_t launch_skinny(const SkinnyProblem &p, cudaStream_t s, int64_t *launches);
// Shared-memory bytes the skinny kernel needs (must be <= 227 KB).
size_t skinny_smem_bytes(int K, int N, size_t esz);

// ---------------------------------------------------------------------------
// MPS transfer chain in one kernel: <bra|ket> bilinear.
// ---------------------------------------------------------------------------
constexpr int kMpsMaxSites = 64, kMpsMaxChi = 32, kMpsMaxD = 4;
struct MpsChain {
  tci_dtype_t dtype;
  int n;
  const void *bra[kMpsMaxSites];
  const void *ket[kMpsMaxSites];
  int d[kMpsMaxSites], bra_r[kMpsMaxSites], ket_r[kMpsMaxSites];   // phys dim, right bonds
  void *out;
  int staged_elems;   // total site elements staged in shared memory (0 = read from global)
};
cudaError_t launch_mps_overlap(const MpsChain &ch, cudaStream_t s, int64_t *launches);

// ---------------------------------------------------------------------------
// Vector kernels (vec.cu) for norm / inner / scale / linear_combine and the
// Lanczos driver. f64 data; complex = (re, im) pairs.
// ---------------------------------------------------------------------------
constexpr int kMaxLC = 8;
// mode 0: out[0] = sum a_i^2 over n_reals; mode 1: complex inner product
// sum conj?(a) b (n_reals = 2 x elements) -> out[0..1]; mode 2: real sum a b.
cudaError_t launch_reduce(int mode, const double *a, const double *b, int64_t n_reals, int conj_a,
                          double *part, double *out, cudaStream_t s, int64_t *launches);
size_t reduce_scratch_bytes();
// several inner products <v_i|w> in one pass over w (bitwise the single ones)
constexpr int kMaxMI = 8, kMaxMIOut = 520;
constexpr int kReduceBlocks = 592;   // reduction CTAs (vec.cu), 4 per SM
cudaError_t launch_multi_inner(bool cplx, const double *const *v, int m, const double *w, int64_t n_reals, int conj_a,
                               double *scratch, double *out, cudaStream_t s, int64_t *launches);
// out[i] = sum_j (cr_j + i ci_j) in_j[i], m <= kMaxLC; out may alias an input
cudaError_t launch_lincomb(bool cplx, const double *const *in, const double *cr, const double *ci, int m,
                           double *out, int64_t n, cudaStream_t s, int64_t *launches);

// offs[i] = sum_l ((i / inner_l) % ext_l) * stride_l over nl legs given
// slowest first (inner_l = product of the extents after l): gamma offsets of
// the GEMM rows / columns for the scatter epilogue
cudaError_t launch_offsets(int64_t *offs, int64_t n, int nl, const int64_t *ext, const int64_t *stride,
                           cudaStream_t s, int64_t *launches);
// the row and column tables of one scatter epilogue in a single launch
cudaError_t launch_offsets2(int64_t *offs1, int64_t n1, int nl1, const int64_t *ext1, const int64_t *stride1,
                            int64_t *offs2, int64_t n2, int nl2, const int64_t *ext2, const int64_t *stride2,
                            cudaStream_t s, int64_t *launches);

// out[r, :] = s[r] * in[r, :] over rows x cols elements (r64 / c128)
cudaError_t launch_row_scale(bool cplx, const double *in, const double *s, double *out, int64_t rows, int64_t cols,
                             cudaStream_t st, int64_t *launches);

// Plain device copy (aliasing fallback) and elementwise helpers.
cudaError_t launch_copy(void *dst, const void *src, size_t bytes, cudaStream_t s, int64_t *launches);
// complex128 conjugation of n elements (in == out allowed)
cudaError_t launch_conj(const void *in, void *out, int64_t n, cudaStream_t s, int64_t *launches);

// ---------------------------------------------------------------------------
// Matrix SVD by block one-sided Jacobi (svd.cu).
// X: npad x ldx working rows (X = A' if I <= J, else A'^H), Y: npad x ldy
// accumulated rotations (Y0 = I). cplx = complex128, else float64.
// ---------------------------------------------------------------------------
struct SvdProblem {
  bool cplx;
  int tall;              // 1: X = A'^H (I > J)
  int64_t n, L;          // rows being orthogonalised (min(I,J)) and their length (max(I,J))
  int64_t npad, ldx;     // n rounded up to 32; L rounded up to 64 (X row pitch)
  int64_t ldy;           // Y row pitch: npad rounded up to 64
  void *X, *Y;
  double *s;             // npad row norms
  unsigned long long *offmax;   // sweep maximum of the off-diagonal measure (double bits)
  unsigned long long *prof = nullptr;   // optional phase clocks (gram, eig, X, Y, rotated pairs)
  // noise floor (squared row norm): rows at or below it are neither rotated
  // nor counted in the convergence measure; their vectors are completed
  double zfloor2 = 0.0;
  // optional per-row flags (npad ints): a pair of two flagged rows is skipped
  // (trunc_svd: both rows below the chi_max cut)
  const int *low = nullptr;
};
size_t svd_round_smem_bytes(bool cplx);
cudaError_t launch_svd_load(const SvdProblem &p, const void *A, int64_t I, int64_t J, cudaStream_t s,
                            int64_t *launches);
// tol: outer convergence (pair skipped when its max relative off-diagonal <= tol);
// tol_in / max_inner: rotation threshold and sweep cap of the 32 x 32 eigensolver
cudaError_t launch_svd_round(const SvdProblem &p, int round, double tol, double tol_in, int max_inner,
                             cudaStream_t s, int64_t *launches);
cudaError_t launch_svd_norms(const SvdProblem &p, cudaStream_t s, int64_t *launches);
cudaError_t launch_svd_gather_rows(bool cplx, void *dst, int64_t ld_dst, const void *src, int64_t ld_src,
                                   const int *perm, const double *s, int64_t nk, int64_t ncols, int conj,
                                   cudaStream_t st, int64_t *launches);
cudaError_t launch_svd_gather_t(bool cplx, void *dst, const void *src, int64_t ld_src, const int *perm,
                                const double *s, int64_t nk, int64_t nr, int conj, cudaStream_t st,
                                int64_t *launches);
// zero rows zl[0..nz) of X -> unit vectors orthogonal to the other selected rows sel[0..nsel)
cudaError_t launch_svd_complete(const SvdProblem &p, const int *sel, int64_t nsel, double *snorm, const int *zl,
                                int nz, cudaStream_t st, int64_t *launches);
cudaError_t launch_svd_gather_s(double *s_out, const double *s, const int *perm, int64_t nk, cudaStream_t st,
                                int64_t *launches);

// Peer-memory all-gather (gather.cu): pointers valid in this
// process (own buffers and the peers' IPC mappings), rank order
constexpr int kMaxRanks = 8;
struct PeerTable {
  void *full[kMaxRanks];    // each rank's full output buffer
  void *flags[kMaxRanks];   // each rank's uint32 flag array [nranks]
};
cudaError_t gather_preload();
cudaError_t ozaki_preload();   // the Ozaki guard's kernels (ozaki.cu)
cudaError_t launch_gather_barrier(const PeerTable &t, int rank, int nranks, uint32_t epoch, int *err,
                                  double timeout_s, cudaStream_t s, int64_t *launches);
cudaError_t launch_push_rows(const void *src, const PeerTable &t, int rank, int nranks, size_t offset_bytes,
                             size_t bytes, cudaStream_t s, int64_t *launches);

}  // namespace tci
