// zipup.cpp -- compressed MPS-MPO application by zip-up (the
// truncated extension of the site-local application of 8(a10); DESIGN.md
// reading R32). The paper has no MPS-MPO algorithm; this is the standard
// left-to-right zip-up built from TCI's own operations: contract
// and trunc_svd.
//
//   C_0[k, a, w] = 1 (all bonds 1)
//   for site i:  T1[k, w, s, b] = sum_a C[k, a, w] A_i[a, s, b]
//                T [k, t, b, v] = sum_{w, s} T1[k, w, s, b] W_i[w, v, s, t]
//                i < n-1: T = U S V^dag at (k t)|(b v), truncated (chi_max, s_min);
//                         B_i = U [k, t, chi'];  C_{i+1} = S V^dag [chi', b, v]
//                i = n-1: B_i = T [k, t, 1]
// Every step runs in the library's kernels (GEMM / thin GEMM / skinny / SVD /
// row scaling); the host loops over sites and keeps the bond bookkeeping.
// The returned trunc_err is the sum over bonds of the discarded weights
// eps_i of the successive truncations.
#include <algorithm>
#include <vector>

#include "runtime.h"

namespace tci {
namespace {

enum { LK = 0, LA = 1, LW = 2, LS = 3, LB = 4, LV = 5, LT = 6 };
const int32_t kLabC[3] = {LK, LA, LW}, kLabA[3] = {LA, LS, LB}, kLabT1[4] = {LK, LW, LS, LB};
const int32_t kLabW[4] = {LW, LV, LS, LT}, kLabT[4] = {LK, LT, LB, LV};

struct ZPlan {
  int n;
  tci_dtype_t dt;
  std::vector<int64_t> chi, D, din, dout, cap;   // chi[i] / D[i]: right bonds of site i; cap[i]: output bond
  size_t off_c, off_t1, off_t, off_s, off_v, off_scr, scr_bytes, total;
};

View mkview(tci_dtype_t dt, std::initializer_list<int64_t> shape, void *data) {
  View v;
  v.dtype = dt;
  v.order = (int)shape.size();
  int k = 0;
  for (int64_t x : shape) v.shape[k++] = x;
  v.data = data;
  return v;
}

tci_status_t zplan(tci_ctx_s *ctx, int n, const tci_tensor_s *const *A, const tci_tensor_s *const *W, int64_t chi_max,
                   ZPlan &p) {
  if (n < 1) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "zipup: need at least one site");
  if (chi_max < 1) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "zipup: chi_max must be >= 1");
  p.n = n;
  p.dt = A[0]->dtype;
  if (p.dt != TCI_R64 && p.dt != TCI_C128) TCI_FAIL(TCI_ERR_UNSUPPORTED, "zipup: dtype must be r64 or c128");
  p.chi.assign(n, 0);
  p.D.assign(n, 0);
  p.din.assign(n, 0);
  p.dout.assign(n, 0);
  p.cap.assign(n, 0);
  int64_t lchi = 1, lD = 1, lcap = 1;
  size_t es = dtype_size(p.dt);
  size_t mc = 0, mt1 = 0, mt = 0, ms = 0, mv = 0, mscr = 0;
  char *fake = reinterpret_cast<char *>(size_t(1) << 40);   // dry runs: distinct, non-overlapping ranges
  for (int i = 0; i < n; i++) {
    const tci_tensor_s *a = A[i], *w = W[i];
    if (a->dtype != p.dt || w->dtype != p.dt) TCI_FAIL(TCI_ERR_UNSUPPORTED, "zipup: dtype mismatch at site %d", i);
    if (a->order != 3 || w->order != 4) TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "zipup: site %d: A order 3, W order 4", i);
    if (a->shape[0] != lchi || w->shape[0] != lD || w->shape[2] != a->shape[1])
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "zipup: bond or physical dimension mismatch at site %d", i);
    p.din[i] = a->shape[1];
    p.dout[i] = w->shape[3];
    p.chi[i] = a->shape[2];
    p.D[i] = w->shape[1];
    if (i == n - 1 && (p.chi[i] != 1 || p.D[i] != 1))
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "zipup: the last site's right bonds must be 1 (open boundary)");
    p.cap[i] = i == n - 1 ? 1 : std::min({chi_max, lcap * p.dout[i], p.chi[i] * p.D[i]});
    // sizes of the carry, T1, T and the SVD outputs at this site
    mc = std::max(mc, (size_t)(lcap * lchi * lD) * es);
    mt1 = std::max(mt1, (size_t)(lcap * lD * p.din[i] * p.chi[i]) * es);
    mt = std::max(mt, (size_t)(lcap * p.dout[i] * p.chi[i] * p.D[i]) * es);
    ms = std::max(ms, (size_t)p.cap[i] * 8);
    mv = std::max(mv, (size_t)(p.cap[i] * p.chi[i] * p.D[i]) * es);
    size_t need = 0;
    const View vc = mkview(p.dt, {lcap, lchi, lD}, fake);
    const View va = view_of(a), vw = view_of(w);
    const View vt1 = mkview(p.dt, {lcap, lD, p.din[i], p.chi[i]}, fake + (size_t(1) << 38));
    const View vt = mkview(p.dt, {lcap, p.dout[i], p.chi[i], p.D[i]}, fake + (size_t(2) << 38));
    tci_status_t st = contract_exec(ctx, vc, kLabC, va, kLabA, vt1, kLabT1, true, &need, nullptr, 0);
    if (st) return st;
    mscr = std::max(mscr, need);
    st = contract_exec(ctx, vt1, kLabT1, vw, kLabW, vt, kLabT, true, &need, nullptr, 0);
    if (st) return st;
    mscr = std::max(mscr, need);
    if (i < n - 1) {
      const int64_t shp[4] = {lcap, p.dout[i], p.chi[i], p.D[i]};
      st = svd_bytes(p.dt, 4, shp, 2, &need);
      if (st) return st;
      mscr = std::max(mscr, need);
    }
    lchi = p.chi[i];
    lD = p.D[i];
    lcap = p.cap[i];
  }
  size_t o = 0;
  p.off_c = o;  o = align_up(o + std::max(mc, es));
  p.off_t1 = o; o = align_up(o + mt1);
  p.off_t = o;  o = align_up(o + mt);
  p.off_s = o;  o = align_up(o + ms);
  p.off_v = o;  o = align_up(o + mv);
  p.off_scr = o;
  p.scr_bytes = mscr;
  p.total = align_up(o + mscr);
  return TCI_OK;
}

}  // namespace

tci_status_t zipup_bytes(tci_ctx_s *ctx, int n, const tci_tensor_s *const *A, const tci_tensor_s *const *W,
                         int64_t chi_max, size_t *bytes) {
  ZPlan p;
  tci_status_t st = zplan(ctx, n, A, W, chi_max, p);
  if (st) return st;
  *bytes = p.total;
  return TCI_OK;
}

tci_status_t zipup_exec(tci_ctx_s *ctx, int n, const tci_tensor_s *const *A, const tci_tensor_s *const *W,
                        tci_tensor_s *const *B, int64_t chi_max, double s_min, double *trunc_err) {
  ZPlan p;
  tci_status_t st = zplan(ctx, n, A, W, chi_max, p);
  if (st) return st;
  if (!(s_min >= 0.0)) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "zipup: s_min must be >= 0");
  // outputs: capacity shapes [cap_{i-1}, dout_i, cap_i]
  int64_t lcap = 1;
  for (int i = 0; i < n; i++) {
    const tci_tensor_s *b = B[i];
    if (b->dtype != p.dt) TCI_FAIL(TCI_ERR_UNSUPPORTED, "zipup: output dtype mismatch at site %d", i);
    if (b->order != 3) TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "zipup: output site %d must be order 3", i);
    if (b->shape[0] != lcap || b->shape[1] != p.dout[i] || b->shape[2] != p.cap[i])
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "zipup: output site %d must have capacity shape [%lld, %lld, %lld]", i,
               (long long)lcap, (long long)p.dout[i], (long long)p.cap[i]);
    lcap = p.cap[i];
  }
  if (ctx->ws_bytes < p.total || (p.total && !ctx->ws))
    TCI_FAIL(TCI_ERR_WORKSPACE, "zipup: workspace %zu B < %zu B (tci_mps_mpo_zipup_workspace_size)", ctx->ws_bytes,
             p.total);
  char *ws = static_cast<char *>(ctx->ws);
  void *Cb = ws + p.off_c, *T1b = ws + p.off_t1, *Tb = ws + p.off_t, *Sb = ws + p.off_s, *Vb = ws + p.off_v;
  void *scr = ws + p.off_scr;
  const bool cplx = p.dt == TCI_C128;
  static const double one[2] = {1.0, 0.0};
  TCI_CUDA_CHECK(cudaMemcpyAsync(Cb, one, cplx ? 16 : 8, cudaMemcpyHostToDevice, ctx->stream));
  int64_t k = 1, lchi = 1, lD = 1;
  double err = 0.0;
  std::vector<int64_t> kept(n, 1);
  for (int i = 0; i < n; i++) {
    size_t need = 0;
    const View vc = mkview(p.dt, {k, lchi, lD}, Cb);
    const View vt1 = mkview(p.dt, {k, lD, p.din[i], p.chi[i]}, T1b);
    const View vt = mkview(p.dt, {k, p.dout[i], p.chi[i], p.D[i]}, Tb);
    st = contract_exec(ctx, vc, kLabC, view_of(A[i]), kLabA, vt1, kLabT1, false, &need, scr, p.scr_bytes);
    if (st) return st;
    st = contract_exec(ctx, vt1, kLabT1, view_of(W[i]), kLabW, vt, kLabT, false, &need, scr, p.scr_bytes);
    if (st) return st;
    if (i == n - 1) {
      TCI_CUDA_CHECK(launch_copy(B[i]->data, Tb, vt.bytes(), ctx->stream, &ctx->launches));
      kept[i] = 1;
      break;
    }
    // T = U S V^dag at (k t) | (b v), truncated
    const int64_t rows = k * p.dout[i], cols = p.chi[i] * p.D[i];
    const int64_t capsvd = std::min(chi_max, std::min(rows, cols));
    tci_tensor_s tu{}, ts{}, tv{};
    for (tci_tensor_s *t : {&tu, &ts, &tv}) {
      t->magic = kTenMagic;
      t->ctx = ctx;
      t->host = false;
    }
    tu.dtype = p.dt; tu.order = 3; tu.shape[0] = k; tu.shape[1] = p.dout[i]; tu.shape[2] = capsvd; tu.data = B[i]->data;
    ts.dtype = TCI_R64; ts.order = 1; ts.shape[0] = capsvd; ts.data = Sb;
    tv.dtype = p.dt; tv.order = 3; tv.shape[0] = capsvd; tv.shape[1] = p.chi[i]; tv.shape[2] = p.D[i]; tv.data = Vb;
    double e = 0.0;
    int64_t chi = 0;
    st = svd_exec(ctx, vt, 2, true, 1, chi_max, 0.0, s_min, &tu, &ts, &tv, &e, &chi, scr, p.scr_bytes);
    if (st) return st;
    err += e;
    kept[i] = chi;
    // carry C = S V^dag [chi, b, v]
    TCI_CUDA_CHECK(launch_row_scale(cplx, static_cast<const double *>(Vb), static_cast<const double *>(Sb),
                                    static_cast<double *>(Cb), chi, cols, ctx->stream, &ctx->launches));
    k = chi;
    lchi = p.chi[i];
    lD = p.D[i];
  }
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  // fold the output descriptors to the kept bonds (metadata; buffers are dense)
  int64_t left = 1;
  for (int i = 0; i < n; i++) {
    B[i]->shape[0] = left;
    B[i]->shape[2] = kept[i];
    left = kept[i];
  }
  if (trunc_err) *trunc_err = err;
  return TCI_OK;
}

}  // namespace tci
