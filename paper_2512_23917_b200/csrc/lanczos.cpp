// lanczos.cpp -- TCI vector functions on device (norm P:1712-1736,
// normalize/scale P:1739-1808, linear_combine P:1980-2010, and the inner
// product used as a full contraction to a scalar) and the Lanczos
// ground-state driver around H_eff.psi (DMRG cited at P:55).
//
// Lanczos (textbook, with full re-orthogonalisation against every stored
// Krylov vector, classical Gram-Schmidt applied twice): v_0 = psi/|psi|;
// w = H v_j; alpha_j = Re<v_j|w>; w -= alpha_j v_j + beta_{j-1} v_{j-1};
// w -= sum_i <v_i|w> v_i (twice); beta_j = |w|; the lowest eigenpair of the
// (j+1)x(j+1) tridiagonal T is found on the host (implicit QL); stop when it
// moved by < tol or beta_j ~ 0; psi <- sum_i y_i v_i (normalised).
// Multi-GPU (8(e)): when the context has a communicator, L is this rank's
// slice L[:, :, b_r]; each H v gives this rank's output slab and one NCCL
// all-gather forms the full w -- the only collective per Lanczos step. All
// vector work is replicated (deterministic kernels), so ranks agree bitwise.
#include <cmath>
#include <cstring>
#include <vector>

#include "runtime.h"

namespace tci {

static tci_status_t vec_check(const View &v) {
  if (v.dtype != TCI_R64 && v.dtype != TCI_C128)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "vector ops: dtype must be r64 or c128");
  return TCI_OK;
}

static int64_t n_reals(const View &v) { return v.size() * (v.dtype == TCI_C128 ? 2 : 1); }

tci_status_t vec_reduce(tci_ctx_s *ctx, int mode, const View &a, const View *b, int conj_a, double out[2]) {
  double *res = static_cast<double *>(ctx->dev_scratch) + (reduce_scratch_bytes() / sizeof(double) - 2);
  double *part = res - 2 * kReduceBlocks;   // the single-reduction partials
  TCI_CUDA_CHECK(launch_reduce(mode, static_cast<const double *>(a.data),
                               b ? static_cast<const double *>(b->data) : nullptr, n_reals(a), conj_a, part,
                               res, ctx->stream, &ctx->launches));
  TCI_CUDA_CHECK(cudaMemcpyAsync(ctx->host_scratch, res, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  out[0] = static_cast<double *>(ctx->host_scratch)[0];
  out[1] = static_cast<double *>(ctx->host_scratch)[1];
  return TCI_OK;
}

tci_status_t vec_norm(tci_ctx_s *ctx, const View &a, double *nrm) {
  tci_status_t st = vec_check(a);
  if (st) return st;
  double r[2];
  st = vec_reduce(ctx, 0, a, nullptr, 0, r);
  if (st) return st;
  *nrm = std::sqrt(r[0]);
  return TCI_OK;
}

tci_status_t vec_inner(tci_ctx_s *ctx, const View &a, const View &b, int conj_a, double out[2]) {
  tci_status_t st = vec_check(a);
  if (st) return st;
  if (a.dtype != b.dtype || a.size() != b.size())
    TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "inner: operands differ in dtype or size");
  return vec_reduce(ctx, a.dtype == TCI_C128 ? 1 : 2, a, &b, conj_a, out);
}

// out[2 i] = <V_i|w> for i < m: one pass over w per kMaxMI vectors, one host
// synchronisation for all (each value bitwise vec_inner's)
static tci_status_t vec_multi_inner(tci_ctx_s *ctx, int m, const View *V, const View &w, int conj_a, double *out) {
  tci_status_t st = vec_check(w);
  if (st) return st;
  std::vector<const double *> vp(m);
  for (int i = 0; i < m; i++) vp[i] = static_cast<const double *>(V[i].data);
  double *scratch = static_cast<double *>(ctx->dev_scratch);
  double *res = scratch + 2 * kReduceBlocks * kMaxMI;
  TCI_CUDA_CHECK(launch_multi_inner(w.dtype == TCI_C128, vp.data(), m, static_cast<const double *>(w.data), n_reals(w),
                                    conj_a, scratch, res, ctx->stream, &ctx->launches));
  TCI_CUDA_CHECK(cudaMemcpyAsync(ctx->host_scratch, res, 2 * m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  memcpy(out, ctx->host_scratch, 2 * m * sizeof(double));
  return TCI_OK;
}

// out = sum_j coef_j in_j (coef as (re, im) pairs); chunks of kMaxLC inputs
tci_status_t vec_lincomb(tci_ctx_s *ctx, int m, const View *ins, const double *coefs, const View &out) {
  tci_status_t st = vec_check(out);
  if (st) return st;
  for (int j = 0; j < m; j++)
    if (ins[j].dtype != out.dtype || ins[j].size() != out.size())
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "linear_combine: inputs must match the output's dtype and size (P:1995)");
  const bool cplx = out.dtype == TCI_C128;
  int j0 = 0;
  bool first = true;
  while (j0 < m || first) {
    const double *in[kMaxLC];
    double cr[kMaxLC], ci[kMaxLC];
    int k = 0;
    if (!first) {   // accumulate onto the running result
      in[k] = static_cast<const double *>(out.data);
      cr[k] = 1.0;
      ci[k] = 0.0;
      k++;
    }
    while (j0 < m && k < kMaxLC) {
      in[k] = static_cast<const double *>(ins[j0].data);
      cr[k] = coefs[2 * j0];
      ci[k] = coefs[2 * j0 + 1];
      k++;
      j0++;
    }
    TCI_CUDA_CHECK(launch_lincomb(cplx, in, cr, ci, k, static_cast<double *>(out.data), out.size(),
                                  ctx->stream, &ctx->launches));
    first = false;
  }
  return TCI_OK;
}

// ---------------------------------------------------------------------------
// symmetric tridiagonal eigenproblem (implicit QL with shifts; eigenvectors)
// ---------------------------------------------------------------------------
static void tqli(std::vector<double> &d, std::vector<double> e, int n, std::vector<double> &z) {
  z.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; i++) z[(size_t)i * n + i] = 1.0;
  for (int i = 1; i < n; i++) e[i - 1] = e[i];
  if (n > 0) e[n - 1] = 0.0;
  for (int l = 0; l < n; l++) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; m++) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 1e-300 + 2.2e-16 * dd) break;
      }
      if (m != l) {
        if (iter++ == 60) break;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0 ? std::fabs(r) : -std::fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; i--) {
          double f = s * e[i], b = c * e[i];
          e[i + 1] = (r = std::hypot(f, g));
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          d[i + 1] = g + (p = s * r);
          g = c * r - b;
          for (int k = 0; k < n; k++) {
            f = z[(size_t)k * n + i + 1];
            z[(size_t)k * n + i + 1] = s * z[(size_t)k * n + i] + c * f;
            z[(size_t)k * n + i] = c * z[(size_t)k * n + i] - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
}

// workspace: heff scratch | w (full) | out slab | V[0..max_iter]
tci_status_t lanczos_bytes(tci_ctx_s *ctx, const View &L, const View &W1, const View &W2, const View &R,
                           const View &psi, int max_iter, size_t *bytes, size_t *heff_b) {
  size_t hb = 0;
  tci_status_t st = heff_plan_bytes(psi.dtype, L.shape[0], L.shape[2], psi.shape[3], R.shape[2], psi.shape[1],
                                    L.shape[1], W1.shape[1], W2.shape[1], &hb, nullptr, ctx->zgemm_algo);
  if (st) return st;
  const size_t vb = align_up(psi.bytes());
  const size_t slab = align_up((size_t)L.shape[2] * psi.shape[1] * psi.shape[2] * R.shape[2] * dtype_size(psi.dtype));
  *heff_b = align_up(hb);
  *bytes = *heff_b + vb + slab + (size_t)(max_iter + 1) * vb;
  (void)W2;
  return TCI_OK;
}

tci_status_t lanczos_exec(tci_ctx_s *ctx, const View &L, const View &W1, const View &W2, const View &R,
                          const View &psi, int max_iter, double tol, double *energy, int *iters) {
  tci_status_t st = vec_check(psi);
  if (st) return st;
  const int P = ctx->nranks;
  if (L.shape[2] * P != psi.shape[0] || R.shape[2] != psi.shape[3])
    TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "lanczos: H_eff must be square (chi_lo x nranks == chi_l, chi_ro == chi_r)");
  if (P > 1 && !ctx->nccl_comm) TCI_FAIL(TCI_ERR_NCCL, "lanczos: sharded run needs tci_comm_init");
  if (max_iter < 1 || max_iter > 512) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "lanczos: max_iter in 1..512");
  size_t need = 0, hb = 0;
  st = lanczos_bytes(ctx, L, W1, W2, R, psi, max_iter, &need, &hb);
  if (st) return st;
  if (need > ctx->ws_bytes || !ctx->ws)
    TCI_FAIL(TCI_ERR_WORKSPACE, "lanczos needs %zu bytes of workspace, %zu attached", need, ctx->ws_bytes);
  char *ws = static_cast<char *>(ctx->ws);
  const size_t vb = align_up(psi.bytes());
  View w = psi, slab = psi;
  w.data = ws + hb;
  slab.shape[0] = L.shape[2];
  slab.data = ws + hb + vb;
  const size_t slab_b = align_up(slab.bytes());
  std::vector<View> V(max_iter + 1, psi);
  for (int i = 0; i <= max_iter; i++) V[i].data = ws + hb + vb + slab_b + (size_t)i * vb;

  // H_eff runs with the heff part of the workspace only
  void *ws_save = ctx->ws;
  const size_t wsb_save = ctx->ws_bytes;
  auto apply_h = [&](const View &x, const View &y) -> tci_status_t {
    ctx->ws = ws;
    ctx->ws_bytes = hb;
    tci_status_t s2 = heff_exec(ctx, L, W1, W2, R, x, P > 1 ? slab : y);
    ctx->ws = ws_save;
    ctx->ws_bytes = wsb_save;
    if (s2) return s2;
    if (P > 1) {
      const int r = nccl_allgather_ptr()(slab.data, y.data, slab.bytes(), 1, ctx->nccl_comm, ctx->stream);
      if (r) TCI_FAIL(TCI_ERR_NCCL, "lanczos: ncclAllGather failed (%d)", r);
    }
    return TCI_OK;
  };
  const bool cplx = psi.dtype == TCI_C128;
  double nrm = 0;
  st = vec_norm(ctx, psi, &nrm);
  if (st) return st;
  if (!(nrm > 0)) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "lanczos: start vector has zero norm");
  {
    const double c[2] = {1.0 / nrm, 0.0};
    st = vec_lincomb(ctx, 1, &psi, c, V[0]);
    if (st) return st;
  }
  std::vector<double> alpha, beta, y;
  double theta = 0, theta_prev = 0;
  int j = 0;
  for (; j < max_iter; j++) {
    st = apply_h(V[j], w);
    if (st) return st;
    // Full re-orthogonalisation by classical Gram-Schmidt against v_0..v_j
    // (its i = j, j-1 terms are the three-term recurrence; alpha_j = <v_j|H v_j>
    // is the first pass's coefficient i = j, bitwise vec_inner's), repeated
    // only when the pass cancelled more than 1 - 1/sqrt(2) of w (Kahan-Parlett
    // "twice is enough", the DGKS criterion; ||w before|| from Pythagoras,
    // no extra read): one pass costs 2j + 5 vector reads / writes.
    double b = 0;
    for (int pass = 0; pass < 2; pass++) {
      std::vector<View> ins(1, w);
      std::vector<double> c = {1.0, 0.0};
      std::vector<double> q(2 * (j + 1));
      st = vec_multi_inner(ctx, j + 1, V.data(), w, 1, q.data());   // all <v_i|w> in one pass over w
      if (st) return st;
      if (pass == 0) alpha.push_back(q[2 * j]);
      double removed = 0;
      for (int i = 0; i <= j; i++) {
        ins.push_back(V[i]);
        c.push_back(-q[2 * i]);
        c.push_back(cplx ? -q[2 * i + 1] : 0.0);
        removed += q[2 * i] * q[2 * i] + q[2 * i + 1] * q[2 * i + 1];
      }
      st = vec_lincomb(ctx, (int)ins.size(), ins.data(), c.data(), w);
      if (st) return st;
      st = vec_norm(ctx, w, &b);
      if (st) return st;
      if (b >= std::sqrt(0.5 * (b * b + removed))) break;   // ||w_after|| >= ||w_before|| / sqrt 2
    }
    beta.push_back(b);
    // lowest Ritz pair of T_{j+1}
    std::vector<double> d(alpha), e(j + 1, 0.0), z;
    for (int i = 1; i <= j; i++) e[i] = beta[i - 1];
    tqli(d, e, j + 1, z);
    int imin = 0;
    for (int i = 1; i <= j; i++)
      if (d[i] < d[imin]) imin = i;
    theta = d[imin];
    y.assign(j + 1, 0.0);
    for (int i = 0; i <= j; i++) y[i] = z[(size_t)i * (j + 1) + imin];
    const bool conv = (j > 0 && std::fabs(theta - theta_prev) < tol) || b < 1e-14 * std::fabs(theta + 1e-300);
    theta_prev = theta;
    if (conv || j + 1 == max_iter) {
      j++;
      break;
    }
    const double c[2] = {1.0 / b, 0.0};
    st = vec_lincomb(ctx, 1, &w, c, V[j + 1]);
    if (st) return st;
  }
  // Ritz vector psi = sum_i y_i v_i, normalised
  {
    std::vector<double> c(2 * j, 0.0);
    for (int i = 0; i < j; i++) c[2 * i] = y[i];
    st = vec_lincomb(ctx, j, V.data(), c.data(), psi);
    if (st) return st;
    double n2 = 0;
    st = vec_norm(ctx, psi, &n2);
    if (st) return st;
    const double s[2] = {1.0 / n2, 0.0};
    st = vec_lincomb(ctx, 1, &psi, s, psi);
    if (st) return st;
  }
  if (energy) *energy = theta;
  if (iters) *iters = j;
  return TCI_OK;
}

}  // namespace tci
