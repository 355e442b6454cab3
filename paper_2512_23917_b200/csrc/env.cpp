// env.cpp -- DMRG environment updates: the step before every
// H_eff in a sweep. With the H_eff conventions of tci_heff_apply (E[ket bond,
// MPO bond, bra bond], W[w_left, w_right, s = ket phys, t = bra phys]):
//   left : out[b,v,e] = sum E[a,w,c] ket[a,s,b] W[w,v,s,t] conj(bra[c,t,e])
//   right: out[a,w,f] = sum ket[a,s,c] W[w,x,s,t] E[c,x,e] conj(bra[f,t,e])
// (R28). Lowered as the H_eff chain is:
//   GEMM (E.ket, contract engine) -> skinny MPO pass (W) -> GEMM (.conj(bra))
// with intermediates laid out so that neither GEMM needs a permute; the
// conjugation (cplx_conj) is one HBM pass over the bra site
// tensor into workspace (~0.3% of the chain at chi = 4096).
#include <algorithm>
#include <cstring>

#include "runtime.h"

namespace tci {
namespace {

enum { EA, EW, EC, ES, EB, ET, EV, EE, NEL };   // label ids (any distinct ints)

struct EnvPlan {
  int64_t chi_k, chi_b, chi_ko, chi_bo, D, Dv, d;   // see env_dims
  View t1, t2, bc;                                   // intermediates (data = offsets until bound)
  size_t off_t1, off_t2, off_bc, off_scr, scr_bytes, total;
  int32_t le[3], lk[3], lt1[4], lt2[4], lb[3], lo[3];
};

// Shapes (left):  E[chi_k, D, chi_b]  ket[chi_k, d, chi_ko]  W[D, Dv, d, d]  bra[chi_b, d, chi_bo]
//                 out[chi_ko, Dv, chi_bo]
// Shapes (right): E[chi_k, D, chi_b]  ket[chi_ko, d, chi_k]  W[Dv, D, d, d]  bra[chi_bo, d, chi_b]
//                 out[chi_ko, Dv, chi_bo]
tci_status_t env_dims(int side, const View &E, const View &K, const View &W, const View &B, const View &O,
                      EnvPlan &p) {
  if (side != 0 && side != 1) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "env: side must be 0 (left) or 1 (right)");
  const tci_dtype_t dt = E.dtype;
  if (K.dtype != dt || W.dtype != dt || B.dtype != dt || O.dtype != dt)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "env: all operands must share one dtype");
  if (dt != TCI_R64 && dt != TCI_C128) TCI_FAIL(TCI_ERR_UNSUPPORTED, "env: dtype must be r64 or c128");
  if (E.order != 3 || K.order != 3 || W.order != 4 || B.order != 3 || O.order != 3)
    TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "env: orders must be E 3, ket 3, W 4, bra 3, out 3");
  p.chi_k = E.shape[0];
  p.D = E.shape[1];
  p.chi_b = E.shape[2];
  p.d = K.shape[1];
  bool ok;
  if (side == 0) {
    p.chi_ko = K.shape[2];
    p.chi_bo = B.shape[2];
    p.Dv = W.shape[1];
    ok = K.shape[0] == p.chi_k && W.shape[0] == p.D && W.shape[2] == p.d && W.shape[3] == p.d &&
         B.shape[0] == p.chi_b && B.shape[1] == p.d;
  } else {
    p.chi_ko = K.shape[0];
    p.chi_bo = B.shape[0];
    p.Dv = W.shape[0];
    ok = K.shape[2] == p.chi_k && W.shape[1] == p.D && W.shape[2] == p.d && W.shape[3] == p.d &&
         B.shape[2] == p.chi_b && B.shape[1] == p.d;
  }
  ok = ok && O.shape[0] == p.chi_ko && O.shape[1] == p.Dv && O.shape[2] == p.chi_bo;
  if (!ok) TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "env: inconsistent shapes (see tci_env_update doc)");
  if (p.D * p.d > kSkinnyMaxK || p.Dv * p.d > kSkinnyMaxN ||
      skinny_smem_bytes((int)(p.D * p.d), (int)(p.Dv * p.d), dtype_size(dt)) > 200 * 1024)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "env: MPO bond x physical dim too large for the skinny pass");
  return TCI_OK;
}

// Plan the chain and its workspace; with ws == nullptr only sizes are computed.
tci_status_t env_plan(tci_ctx_s *ctx, int side, const View &E, const View &K, const View &W, const View &B,
                      const View &O, EnvPlan &p) {
  tci_status_t st = env_dims(side, E, K, W, B, O, p);
  if (st) return st;
  const tci_dtype_t dt = E.dtype;
  auto mk = [&](View &v, std::initializer_list<int64_t> shp) {
    v = View{};
    v.dtype = dt;
    v.order = (int)shp.size();
    int k = 0;
    for (int64_t s : shp) v.shape[k++] = s;
  };
  if (side == 0) {
    // T1[w,c,s,b] = sum_a E[a,w,c] ket[a,s,b];  T2[c,t,b,v] = sum_{w,s} T1 W[w,v,s,t]
    mk(p.t1, {p.D, p.chi_b, p.d, p.chi_ko});
    mk(p.t2, {p.chi_b, p.d, p.chi_ko, p.Dv});
    mk(p.bc, {p.chi_b, p.d, p.chi_bo});
    const int32_t le[3] = {EA, EW, EC}, lk[3] = {EA, ES, EB}, lt1[4] = {EW, EC, ES, EB},
                  lt2[4] = {EC, ET, EB, EV}, lb[3] = {EC, ET, EE}, lo[3] = {EB, EV, EE};
    memcpy(p.le, le, sizeof le); memcpy(p.lk, lk, sizeof lk); memcpy(p.lt1, lt1, sizeof lt1);
    memcpy(p.lt2, lt2, sizeof lt2); memcpy(p.lb, lb, sizeof lb); memcpy(p.lo, lo, sizeof lo);
  } else {
    // T1[a,s,x,e] = sum_c ket[a,s,c] E[c,x,e];  T2[a,w,t,e] = sum_{s,x} T1 W[w,x,s,t]
    mk(p.t1, {p.chi_ko, p.d, p.D, p.chi_b});
    mk(p.t2, {p.chi_ko, p.Dv, p.d, p.chi_b});
    mk(p.bc, {p.chi_bo, p.d, p.chi_b});
    // here EC = ket right bond c, EW = x (E's MPO bond), EE = e (E's bra bond),
    // EA = a, ES = s, EV = w (out MPO bond), ET = t, EB = f (out bra bond)
    const int32_t le[3] = {EC, EW, EE}, lk[3] = {EA, ES, EC}, lt1[4] = {EA, ES, EW, EE},
                  lt2[4] = {EA, EV, ET, EE}, lb[3] = {EB, ET, EE}, lo[3] = {EA, EV, EB};
    memcpy(p.le, le, sizeof le); memcpy(p.lk, lk, sizeof lk); memcpy(p.lt1, lt1, sizeof lt1);
    memcpy(p.lt2, lt2, sizeof lt2); memcpy(p.lb, lb, sizeof lb); memcpy(p.lo, lo, sizeof lo);
  }
  const bool cplx = dt == TCI_C128;
  size_t off = 0;
  p.off_t1 = off;
  off = align_up(off + p.t1.bytes());
  p.off_t2 = off;
  off = align_up(off + p.t2.bytes());
  p.off_bc = off;
  off = align_up(off + (cplx ? p.bc.bytes() : 0));
  p.off_scr = off;
  // scratch of the two GEMMs (contract engine dry runs; intermediates are 256-byte aligned)
  View t1 = p.t1, t2 = p.t2, bc = cplx ? p.bc : B;
  t1.data = t2.data = reinterpret_cast<void *>(256);
  if (cplx) bc.data = reinterpret_cast<void *>(256);
  size_t n1 = 0, n2 = 0;
  const View &e1 = side == 0 ? E : K, &k1 = side == 0 ? K : E;
  const int32_t *l1a = side == 0 ? p.le : p.lk, *l1b = side == 0 ? p.lk : p.le;
  st = contract_exec(ctx, e1, l1a, k1, l1b, t1, p.lt1, true, &n1, nullptr, 0);
  if (st) return st;
  st = contract_exec(ctx, t2, p.lt2, bc, p.lb, O, p.lo, true, &n2, nullptr, 0);
  if (st) return st;
  p.scr_bytes = align_up(std::max(n1, n2));
  p.total = off + p.scr_bytes;
  return TCI_OK;
}

}  // namespace

tci_status_t env_bytes(tci_ctx_s *ctx, int side, const View &E, const View &K, const View &W, const View &B,
                       const View &O, size_t *bytes) {
  EnvPlan p{};
  tci_status_t st = env_plan(ctx, side, E, K, W, B, O, p);
  if (st) return st;
  *bytes = p.total;
  return TCI_OK;
}

tci_status_t env_exec(tci_ctx_s *ctx, int side, const View &E, const View &K, const View &W, const View &B,
                      const View &O) {
  EnvPlan p{};
  tci_status_t st = env_plan(ctx, side, E, K, W, B, O, p);
  if (st) return st;
  if (p.total > ctx->ws_bytes || (p.total && !ctx->ws))
    TCI_FAIL(TCI_ERR_WORKSPACE, "env needs %zu bytes of workspace, %zu attached", p.total, ctx->ws_bytes);
  char *ws = static_cast<char *>(ctx->ws);
  const tci_dtype_t dt = E.dtype;
  View t1 = p.t1, t2 = p.t2, bc = B;
  t1.data = ws + p.off_t1;
  t2.data = ws + p.off_t2;
  // ---- conj(bra) into workspace (complex only) ----
  if (dt == TCI_C128) {
    bc = p.bc;
    bc.data = ws + p.off_bc;
    int64_t n = 1;
    for (int k = 0; k < 3; k++) n *= B.shape[k];
    TCI_CUDA_CHECK(launch_conj(B.data, bc.data, n, ctx->stream, &ctx->launches));
  }
  // ---- GEMM1 ----
  size_t need = 0;
  if (side == 0)
    st = contract_exec(ctx, E, p.le, K, p.lk, t1, p.lt1, false, &need, ws + p.off_scr, p.scr_bytes);
  else
    st = contract_exec(ctx, K, p.lk, E, p.le, t1, p.lt1, false, &need, ws + p.off_scr, p.scr_bytes);
  if (st) return st;
  // ---- skinny MPO pass ----
  const int64_t d = p.d, D = p.D, Dv = p.Dv;
  SkinnyProblem sp{};
  sp.dtype = dt;
  sp.in = t1.data;
  sp.W = W.data;
  sp.out = t2.data;
  if (side == 0) {
    // T2[c,t,b,v] = sum_{w,s} T1[w,c,s,b] W[w,v,s,t]; batches (c, b), b unit-stride in T1
    const int64_t cb = p.chi_b, ck = p.chi_ko;
    sp.nb[0] = 1; sp.nb[1] = cb; sp.nb[2] = ck;
    sp.in_sb[0] = 0; sp.in_sb[1] = d * ck; sp.in_sb[2] = 1;
    sp.out_sb[0] = 0; sp.out_sb[1] = d * ck * Dv; sp.out_sb[2] = Dv;
    sp.K = (int)(D * d); sp.N = (int)(d * Dv);
    sp.k_lo = 1; sp.n_lo = (int)Dv;
    int k = 0;
    for (int64_t w = 0; w < D; w++)
      for (int64_t s = 0; s < d; s++, k++) {
        sp.in_koff[k] = w * cb * d * ck + s * ck;
        sp.w_koff[k] = (int32_t)(w * Dv * d * d + s * d);
      }
    int n = 0;
    for (int64_t t = 0; t < d; t++)
      for (int64_t v = 0; v < Dv; v++, n++) {
        sp.out_noff[n] = t * ck * Dv + v;
        sp.w_noff[n] = (int32_t)(v * d * d + t);
      }
  } else {
    // T2[a,w,t,e] = sum_{s,x} T1[a,s,x,e] W[w,x,s,t]; batches (a, e), e unit-stride in T1
    const int64_t ca = p.chi_ko, ce = p.chi_b;
    sp.nb[0] = 1; sp.nb[1] = ca; sp.nb[2] = ce;
    sp.in_sb[0] = 0; sp.in_sb[1] = d * D * ce; sp.in_sb[2] = 1;
    sp.out_sb[0] = 0; sp.out_sb[1] = Dv * d * ce; sp.out_sb[2] = 1;
    sp.K = (int)(d * D); sp.N = (int)(Dv * d);
    sp.k_lo = 1; sp.n_lo = 1;
    int k = 0;
    for (int64_t s = 0; s < d; s++)
      for (int64_t x = 0; x < D; x++, k++) {
        sp.in_koff[k] = s * D * ce + x * ce;
        sp.w_koff[k] = (int32_t)(x * d * d + s * d);
      }
    int n = 0;
    for (int64_t w = 0; w < Dv; w++)
      for (int64_t t = 0; t < d; t++, n++) {
        sp.out_noff[n] = w * d * ce + t * ce;
        sp.w_noff[n] = (int32_t)(w * D * d * d + t);
      }
  }
  st = run_skinny(ctx, sp);
  if (st) return st;
  // ---- GEMM2: out = T2 . conj(bra) ----
  return contract_exec(ctx, t2, p.lt2, bc, p.lb, O, p.lo, false, &need, ws + p.off_scr, p.scr_bytes);
}

}  // namespace tci
