// chains.cpp -- the contraction chains of the north star (SURVEY 8(a7),
// 8(a8)): two-site H_eff.psi with its FLOP-count order planner, and the TEBD
// gate application theta = (A.B).U. Definitions: DESIGN.md R15, R16 (the
// paper defines neither; DMRG is cited at PAPER.md:55, iTEBD is Application A,
// PAPER.md:392-403).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "runtime.h"

namespace tci {

// ---------------------------------------------------------------------------
// H_eff order planner: exhaustive search over pairwise contraction trees of
// the five tensors {L, psi, W1, W2, R} by multiply-add count (dynamic
// programming over subsets; every binary tree is considered), ties broken by
// the largest intermediate, then by a fixed canonical order (lowest subset
// mask first). Labels: L(a,w,b) psi(a,s,t,c) W1(w,v,s,p) W2(v,x,t,q) R(c,x,e),
// output (b,p,q,e).
// ---------------------------------------------------------------------------
namespace {

enum { LA, LW, LB, LS, LT, LC, LV, LP, LX, LQ, LE, NLAB };
const int kTen[5][4] = {{LA, LW, LB, -1}, {LA, LS, LT, LC}, {LW, LV, LS, LP},
                        {LV, LX, LT, LQ}, {LC, LX, LE, -1}};
const int kOut[4] = {LB, LP, LQ, LE};

struct Node {
  double cost = -1, peak = 0;
  int left = 0;   // submask of the first child (0 = leaf)
  uint32_t labels = 0;
};

uint32_t labels_of_mask(int mask) {
  uint32_t inside = 0, outside = 0;
  for (int t = 0; t < 5; t++)
    for (int k = 0; k < 4; k++)
      if (kTen[t][k] >= 0) ((mask >> t) & 1 ? inside : outside) |= 1u << kTen[t][k];
  uint32_t out = 0;
  for (int k = 0; k < 4; k++) out |= 1u << kOut[k];
  return inside & (outside | out);
}

}  // namespace

// Returns the optimal tree as a string like "((((L.psi).W1).W2).R)" and its
// MAC count; used by the executor and reported by tci_heff_plan (tests).
static std::string tree_str(const std::vector<Node> &nd, int mask) {
  static const char *names[5] = {"L", "psi", "W1", "W2", "R"};
  if (__builtin_popcount(mask) == 1) return names[__builtin_ctz(mask)];
  return "(" + tree_str(nd, nd[mask].left) + "." + tree_str(nd, mask ^ nd[mask].left) + ")";
}

static std::vector<Node> plan_heff_tree(const int64_t dims[NLAB]) {
  std::vector<Node> nd(32);
  for (int t = 0; t < 5; t++) {
    nd[1 << t].cost = 0;
    nd[1 << t].labels = labels_of_mask(1 << t);
  }
  for (int mask = 1; mask < 32; mask++) {
    if (__builtin_popcount(mask) < 2) continue;
    nd[mask].labels = labels_of_mask(mask);
    for (int sub = (mask - 1) & mask; sub > 0; sub = (sub - 1) & mask) {
      const int other = mask ^ sub;
      if (sub > other) continue;   // unordered pairs, canonical: lower mask first
      const Node &x = nd[sub], &y = nd[other];
      if (x.cost < 0 || y.cost < 0) continue;
      double macs = 1, size = 1;
      const uint32_t all = x.labels | y.labels;
      for (int l = 0; l < NLAB; l++) {
        if (all >> l & 1) macs *= (double)dims[l];
        if (nd[mask].labels >> l & 1) size *= (double)dims[l];
      }
      const double cost = x.cost + y.cost + macs;
      const double peak = std::max({x.peak, y.peak, size});
      Node &z = nd[mask];
      if (z.cost < 0 || cost < z.cost || (cost == z.cost && peak < z.peak)) {
        z.cost = cost;
        z.peak = peak;
        z.left = sub;
      }
    }
  }
  return nd;
}

// Executor fast path: the tree (((L.psi).W1).W2).R or ((L.psi).(W1.W2)).R.
static bool is_standard_tree(const std::vector<Node> &nd) {
  const std::string s = tree_str(nd, 31);
  return s == "((((L.psi).W1).W2).R)" || s == "(((L.psi).(W1.W2)).R)" ||
         s == "(R.(((L.psi).W1).W2))" || s == "(R.((L.psi).(W1.W2)))";
}

namespace {
struct HeffDims {
  int64_t chi_l, chi_lo, chi_r, chi_ro, d, D, D1, D2;
};
struct HeffLayout {
  bool fused;
  size_t es, t1, t2, t3, w12, w12_scratch, off_x, off_y, off_w12, off_w12s, total;
};

// time model (seconds) used only to choose fused vs two-step MPO passes
double pass_time(double bytes, double macs, bool cplx) {
  const double hbm = 6.4e12, fp64 = 36.0e12;
  return std::max(bytes / hbm, macs * (cplx ? 8.0 : 2.0) / fp64);
}

HeffLayout heff_layout(const HeffDims &h, tci_dtype_t dt) {
  HeffLayout L{};
  L.es = dtype_size(dt);
  const bool cplx = dtype_is_complex(dt);
  const size_t es = L.es;
  const double bc = (double)h.chi_lo * h.chi_r;
  L.t1 = (size_t)(h.D * h.chi_lo * h.d * h.d * h.chi_r) * es;
  L.t2 = (size_t)(h.chi_lo * h.d * h.D1 * h.d * h.chi_r) * es;
  L.t3 = (size_t)(h.chi_lo * h.d * h.d * h.chi_r * h.D2) * es;
  const int Kf = (int)(h.D * h.d * h.d), Nf = (int)(h.D2 * h.d * h.d);
  const bool fused_ok = Kf <= kSkinnyMaxK && Nf <= kSkinnyMaxN &&
                        skinny_smem_bytes(Kf, Nf, es) <= 200 * 1024;
  const double t_fused = pass_time((double)(L.t1 + L.t3), bc * Kf * Nf, cplx);
  const double t_two = pass_time((double)(L.t1 + L.t2), bc * h.d * (h.D * h.d) * (h.D1 * h.d), cplx) +
                       pass_time((double)(L.t2 + L.t3), bc * h.d * (h.D1 * h.d) * (h.D2 * h.d), cplx);
  const bool two_ok = h.D * h.d <= kSkinnyMaxK && h.D1 * h.d <= kSkinnyMaxN &&
                      h.D2 * h.d <= kSkinnyMaxN && skinny_smem_bytes((int)(h.D * h.d), (int)(h.D1 * h.d), es) <= 200 * 1024 &&
                      skinny_smem_bytes((int)(h.D1 * h.d), (int)(h.D2 * h.d), es) <= 200 * 1024;
  L.fused = fused_ok && (!two_ok || t_fused <= t_two);
  L.w12 = L.fused ? (size_t)(h.D * h.d * h.d * h.D2 * h.d * h.d) * es : 0;
  // W12 = contract(W1 "wvsp", W2 "vxtq" -> "wspxtq"): W1 is permuted to
  // [w,s,p,v] in scratch (the only non-blocked operand)
  L.w12_scratch = L.fused ? align_up((size_t)(h.D * h.D1 * h.d * h.d) * es) : 0;
  size_t off = 0;
  L.off_x = off;
  off = align_up(off + (L.fused ? L.t1 : std::max(L.t1, L.t3)));
  L.off_y = off;
  off = align_up(off + (L.fused ? L.t3 : L.t2));
  L.off_w12 = off;
  off = align_up(off + L.w12);
  L.off_w12s = off;
  off = align_up(off + L.w12_scratch);
  L.total = off;
  return L;
}
}  // namespace

// Ozaki scratch for the two chain GEMMs (0 when not used)
static size_t heff_ozaki_bytes(tci_dtype_t dt, int zalgo, int64_t chi_l, int64_t chi_lo, int64_t chi_r,
                               int64_t chi_ro, int64_t d, int64_t D, int64_t D2) {
  if ((dt != TCI_C128 && dt != TCI_R64) || zalgo != kZOzaki) return 0;   // r64: real Ozaki-II
  size_t b = 0;
  const int64_t M1 = D * chi_lo, N1 = d * d * chi_r, K1 = chi_l;
  if (ozaki_worthwhile(M1, N1, K1, dt)) b = std::max(b, ozaki_workspace_bytes(M1, N1, K1));
  const int64_t M4 = chi_lo * d * d, N4 = chi_ro, K4 = chi_r * D2;
  if (ozaki_worthwhile(M4, N4, K4, dt)) b = std::max(b, ozaki_workspace_bytes(M4, N4, K4));
  return b ? align_up(b) : 0;
}

tci_status_t heff_plan_bytes(tci_dtype_t dt, int64_t chi_l, int64_t chi_lo, int64_t chi_r,
                             int64_t chi_ro, int64_t d, int64_t D, int64_t D1, int64_t D2,
                             size_t *bytes, bool *fused_w12, int zalgo) {
  if (dt != TCI_R64 && dt != TCI_C128) TCI_FAIL(TCI_ERR_UNSUPPORTED, "heff: dtype must be r64 or c128");
  if (chi_l < 1 || chi_lo < 1 || chi_r < 1 || chi_ro < 1 || d < 1 || D < 1 || D1 < 1 || D2 < 1)
    TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "heff: dimension < 1");
  HeffDims h{chi_l, chi_lo, chi_r, chi_ro, d, D, D1, D2};
  HeffLayout L = heff_layout(h, dt);
  const int64_t dims[NLAB] = {chi_l, D, chi_lo, d, d, chi_r, D1, d, D2, d, chi_ro};
  std::vector<Node> nd = plan_heff_tree(dims);
  size_t need = L.total + heff_ozaki_bytes(dt, zalgo, chi_l, chi_lo, chi_r, chi_ro, d, D, D2);
  if (!is_standard_tree(nd)) {
    // generic tree executor: every intermediate + the largest contract scratch
    // (bounded by 3x the largest intermediate) -- computed in heff_exec
    need = 0;
    double big = 0;
    for (int m = 1; m < 31; m++)
      if (__builtin_popcount(m) >= 2) {
        double s = 1;
        for (int l = 0; l < NLAB; l++)
          if (nd[m].labels >> l & 1) s *= (double)dims[l];
        big = std::max(big, s);
      }
    need = align_up((size_t)(big * dtype_size(dt))) * 6;
  }
  if (bytes) *bytes = need;
  if (fused_w12) *fused_w12 = L.fused;
  return TCI_OK;
}

// generic tree execution through contract_exec (used only when the
// FLOP-optimal tree is not the standard L-first chain, e.g. chi_l >> chi_r)
static tci_status_t exec_tree(tci_ctx_s *ctx, const std::vector<Node> &nd, int mask,
                              const View *leaf, const int64_t dims[NLAB], char *&arena,
                              size_t &left, View &out, std::vector<int32_t> &labs) {
  if (__builtin_popcount(mask) == 1) {
    const int t = __builtin_ctz(mask);
    out = leaf[t];
    labs.clear();
    for (int k = 0; k < 4; k++)
      if (kTen[t][k] >= 0) labs.push_back(kTen[t][k]);
    return TCI_OK;
  }
  View x, y;
  std::vector<int32_t> lx, ly;
  tci_status_t st = exec_tree(ctx, nd, nd[mask].left, leaf, dims, arena, left, x, lx);
  if (st) return st;
  st = exec_tree(ctx, nd, mask ^ nd[mask].left, leaf, dims, arena, left, y, ly);
  if (st) return st;
  // result labels: those of x then y that survive, natural order
  labs.clear();
  const uint32_t keep = nd[mask].labels;
  for (int32_t l : lx)
    if (keep >> l & 1) labs.push_back(l);
  for (int32_t l : ly)
    if ((keep >> l & 1) && std::find(labs.begin(), labs.end(), l) == labs.end()) labs.push_back(l);
  if (mask == 31) {
    // final: write into `out` (already the user's tensor) in (b,p,q,e) order
    labs.assign(kOut, kOut + 4);
  } else {
    View r;
    r.dtype = x.dtype;
    r.order = (int)labs.size();
    for (int k = 0; k < r.order; k++) r.shape[k] = dims[labs[k]];
    const size_t bytes = align_up(r.bytes());
    if (bytes > left) TCI_FAIL(TCI_ERR_WORKSPACE, "heff: workspace too small (generic tree)");
    r.data = arena;
    arena += bytes;
    left -= bytes;
    out = r;
  }
  size_t need = 0;
  st = contract_exec(ctx, x, lx.data(), y, ly.data(), out, labs.data(), true, &need, nullptr, 0);
  if (st) return st;
  if (need > left) TCI_FAIL(TCI_ERR_WORKSPACE, "heff: workspace too small (generic tree)");
  return contract_exec(ctx, x, lx.data(), y, ly.data(), out, labs.data(), false, &need, arena, left);
}

namespace {
// GEMM4 row chunk finished (enqueued) on the context stream: copy it out
void stage_rows_out(void *user, int64_t m0, int64_t mc) {
  HeffStaging *st = static_cast<HeffStaging *>(user);
  if (st->err != cudaSuccess || !st->out_host) return;   // no host twin: the result stays on the device
  tci_ctx_s *ctx = st->ctx;
  cudaError_t e = cudaEventRecord(st->ev_rows, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->copy_stream, st->ev_rows, 0);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(st->out_host + m0 * st->row_bytes, st->out_dev + m0 * st->row_bytes, mc * st->row_bytes,
                        cudaMemcpyDeviceToHost, ctx->copy_stream);
  st->err = e;
}
// GEMM1 is about to read A rows (w b) [m0, m0 + mc) = L columns: copy that
// column block in on the copy stream and make the context stream wait for it
void stage_L_in(void *user, int64_t m0, int64_t mc) {
  HeffStaging *st = static_cast<HeffStaging *>(user);
  if (st->err != cudaSuccess) return;
  tci_ctx_s *ctx = st->ctx;
  const size_t pitch = (size_t)st->L_cols * st->es;
  cudaError_t e = cudaMemcpy2DAsync(st->L_dev + m0 * st->es, pitch, st->L_host + m0 * st->es, pitch,
                                    (size_t)mc * st->es, (size_t)st->L_rows, cudaMemcpyDefault, ctx->copy_stream);
  if (e == cudaSuccess) e = cudaEventRecord(st->ev_L, ctx->copy_stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->stream, st->ev_L, 0);
  st->err = e;
}
}  // namespace

tci_status_t heff_exec(tci_ctx_s *ctx, const View &L, const View &W1, const View &W2, const View &R,
                       const View &psi, const View &out, HeffStaging *stage, HeffGather *gather) {
  if (gather) gather->fused = false;
  const tci_dtype_t dt = L.dtype;
  if (W1.dtype != dt || W2.dtype != dt || R.dtype != dt || psi.dtype != dt || out.dtype != dt)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "heff: all operands must share one dtype");
  if (dt != TCI_R64 && dt != TCI_C128) TCI_FAIL(TCI_ERR_UNSUPPORTED, "heff: dtype must be r64 or c128");
  if (L.order != 3 || W1.order != 4 || W2.order != 4 || R.order != 3 || psi.order != 4 || out.order != 4)
    TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "heff: orders must be L 3, W1 4, W2 4, R 3, psi 4, out 4");
  HeffDims h{L.shape[0], L.shape[2], psi.shape[3], R.shape[2], psi.shape[1], L.shape[1], W1.shape[1],
             W2.shape[1]};
  const bool ok = psi.shape[0] == h.chi_l && psi.shape[2] == h.d && W1.shape[0] == h.D &&
                  W1.shape[2] == h.d && W1.shape[3] == h.d && W2.shape[0] == h.D1 &&
                  W2.shape[2] == h.d && W2.shape[3] == h.d && R.shape[0] == h.chi_r &&
                  R.shape[1] == h.D2 && out.shape[0] == h.chi_lo && out.shape[1] == h.d &&
                  out.shape[2] == h.d && out.shape[3] == h.chi_ro;
  if (!ok) TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "heff: inconsistent shapes (see tci_heff_apply doc)");
  size_t need = 0;
  bool fused = false;
  tci_status_t st = heff_plan_bytes(dt, h.chi_l, h.chi_lo, h.chi_r, h.chi_ro, h.d, h.D, h.D1, h.D2,
                                    &need, &fused, ctx->zgemm_algo);
  if (st) return st;
  if (need > ctx->ws_bytes || (need && !ctx->ws))
    TCI_FAIL(TCI_ERR_WORKSPACE, "heff needs %zu bytes of workspace, %zu attached", need, ctx->ws_bytes);
  const int64_t dims[NLAB] = {h.chi_l, h.D, h.chi_lo, h.d, h.d, h.chi_r, h.D1, h.d, h.D2, h.d, h.chi_ro};
  std::vector<Node> nd = plan_heff_tree(dims);
  char *ws = static_cast<char *>(ctx->ws);
  if (stage) TCI_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, stage->ev_in, 0));
  // R's H2D follows L's on the copy stream
  auto copy_R = [&]() -> tci_status_t {
    TCI_CUDA_CHECK(cudaMemcpyAsync(stage->R_dev, stage->R_host, stage->R_bytes, cudaMemcpyDefault,
                                   ctx->copy_stream));
    TCI_CUDA_CHECK(cudaEventRecord(stage->ev_R, ctx->copy_stream));
    return TCI_OK;
  };
  if (!is_standard_tree(nd)) {
    if (stage) {
      stage_L_in(stage, 0, stage->L_cols);
      TCI_CUDA_CHECK(stage->err);
      st = copy_R();
      if (st) return st;
      TCI_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, stage->ev_R, 0));
    }
    const View leaf[5] = {L, psi, W1, W2, R};
    char *arena = ws;
    size_t left = ctx->ws_bytes;
    View o = out;
    std::vector<int32_t> labs;
    st = exec_tree(ctx, nd, 31, leaf, dims, arena, left, o, labs);
    if (st || !stage) return st;
    stage_rows_out(stage, 0, out.shape[0] * out.shape[1] * out.shape[2]);
    TCI_CUDA_CHECK(stage->err);
    return TCI_OK;
  }
  const HeffLayout lay = heff_layout(h, dt);
  const int64_t d = h.d, chi_lo = h.chi_lo, chi_r = h.chi_r;
  const size_t oz_b = heff_ozaki_bytes(dt, ctx->zgemm_algo, h.chi_l, h.chi_lo, h.chi_r, h.chi_ro, h.d, h.D, h.D2);
  auto set_zalgo = [&](GemmProblem &g) {
    g.zalgo = ctx->zgemm_algo == kZOzaki ? kZ3M : ctx->zgemm_algo;
    // (the real Ozaki GEMM takes its row exponents up front: not with staged input)
    if (oz_b && ozaki_worthwhile(g.M, g.N, g.K, g.dtype) && !(dt == TCI_R64 && stage)) {
      g.zalgo = kZOzaki;
      g.oz_ws = ws + lay.total;
      g.oz_ws_bytes = oz_b;
    }
  };
  void *T1 = ws + lay.off_x;
  // ---- GEMM1: T1[w,b,s,t,c] = sum_a L[a,w,b] psi[a,s,t,c] ----
  {
    GemmProblem g{};
    g.dtype = dt;
    g.M = h.D * chi_lo; g.K = h.chi_l; g.N = d * d * chi_r;
    g.A = L.data; g.a_sm = 1; g.a_sk = g.M;
    g.B = psi.data; g.b_sk = g.N; g.b_sn = 1;
    g.C = T1; g.c_sm = g.N;
    set_zalgo(g);
    if (g.K == 1) g.a_sk = 0;
    if (g.M == 1) { g.a_sm = 1; g.a_sk = 1; }
    if (g.K == 1 && g.N == 1) g.b_sk = 1;
    else if (g.K == 1) g.b_sk = 0;
    if (stage && g.zalgo == kZOzaki && g.a_sm == 1) {
      // L arrives column block by column block while GEMM1 computes
      g.rows_needed = stage_L_in;
      g.rows_user = stage;
      g.max_chunk_rows = std::max<int64_t>(256, (g.M + 7) / 8);
      { tci_status_t _r = run_gemm(ctx, g); if (_r) return _r; }
      TCI_CUDA_CHECK(stage->err);
    } else if (stage && g.a_sm == 1 && g.M >= 1024) {
      const int64_t M = g.M, ch = (M + 3) / 4;
      for (int64_t m0 = 0; m0 < M; m0 += ch) {
        GemmProblem gc = g;
        gc.M = std::min(ch, M - m0);
        gc.A = static_cast<const char *>(g.A) + m0 * dtype_size(dt);
        gc.C = static_cast<char *>(g.C) + m0 * g.c_sm * dtype_size(dt);
        if (gc.zalgo == kZOzaki && !ozaki_worthwhile(gc.M, gc.N, gc.K, gc.dtype)) gc.zalgo = kZ3M;
        stage_L_in(stage, m0, gc.M);
        TCI_CUDA_CHECK(stage->err);
        { tci_status_t _r = run_gemm(ctx, gc); if (_r) return _r; }
      }
    } else {
      if (stage) {
        stage_L_in(stage, 0, stage->L_cols);
        TCI_CUDA_CHECK(stage->err);
      }
      tci_status_t _r = run_gemm(ctx, g);
      if (_r) return _r;
    }
    if (stage) {
      st = copy_R();
      if (st) return st;
    }
  }
  void *T3;
  if (lay.fused) {
    // ---- W12[w,s,p,x,t,q] = sum_v W1[w,v,s,p] W2[v,x,t,q] ----
    View w12;
    w12.dtype = dt;
    w12.order = 6;
    const int64_t shp[6] = {h.D, d, d, h.D2, d, d};
    for (int k = 0; k < 6; k++) w12.shape[k] = shp[k];
    w12.data = ws + lay.off_w12;
    const int32_t l1[4] = {LW, LV, LS, LP}, l2[4] = {LV, LX, LT, LQ}, l12[6] = {LW, LS, LP, LX, LT, LQ};
    size_t n2 = 0;
    st = contract_exec(ctx, W1, l1, W2, l2, w12, l12, true, &n2, nullptr, 0);
    if (st) return st;
    st = contract_exec(ctx, W1, l1, W2, l2, w12, l12, false, &n2, ws + lay.off_w12s, lay.w12_scratch);
    if (st) return st;
    // ---- T3[b,p,q,c,x] = sum_{w,s,t} T1[w,b,s,t,c] W12[w,s,p,x,t,q] ----
    T3 = ws + lay.off_y;
    SkinnyProblem sp{};
    sp.dtype = dt;
    sp.nb[0] = 1; sp.nb[1] = chi_lo; sp.nb[2] = chi_r;
    sp.in_sb[0] = 0; sp.in_sb[1] = d * d * chi_r; sp.in_sb[2] = 1;
    sp.out_sb[0] = 0; sp.out_sb[1] = d * d * chi_r * h.D2; sp.out_sb[2] = h.D2;
    sp.K = (int)(h.D * d * d); sp.N = (int)(d * d * h.D2);
    sp.k_lo = 1; sp.n_lo = (int)h.D2;
    sp.in = T1; sp.W = w12.data; sp.out = T3;
    const int64_t w12s[6] = {d * d * h.D2 * d * d, d * h.D2 * d * d, h.D2 * d * d, d * d, d, 1};
    int k = 0;
    for (int64_t w = 0; w < h.D; w++)
      for (int64_t s = 0; s < d; s++)
        for (int64_t t = 0; t < d; t++, k++) {
          sp.in_koff[k] = w * chi_lo * d * d * chi_r + s * d * chi_r + t * chi_r;
          sp.w_koff[k] = (int32_t)(w * w12s[0] + s * w12s[1] + t * w12s[4]);
        }
    int n = 0;
    for (int64_t p = 0; p < d; p++)
      for (int64_t q = 0; q < d; q++)
        for (int64_t x = 0; x < h.D2; x++, n++) {
          sp.out_noff[n] = p * d * chi_r * h.D2 + q * chi_r * h.D2 + x;
          sp.w_noff[n] = (int32_t)(p * w12s[2] + x * w12s[3] + q * w12s[5]);
        }
    { tci_status_t _r = run_skinny(ctx, sp); if (_r) return _r; }
  } else {
    // ---- T2[b,t,v,p,c] = sum_{w,s} T1[w,b,s,t,c] W1[w,v,s,p] ----
    void *T2 = ws + lay.off_y;
    {
      SkinnyProblem sp{};
      sp.dtype = dt;
      sp.nb[0] = chi_lo; sp.nb[1] = d; sp.nb[2] = chi_r;
      sp.in_sb[0] = d * d * chi_r; sp.in_sb[1] = chi_r; sp.in_sb[2] = 1;
      sp.out_sb[0] = d * h.D1 * d * chi_r; sp.out_sb[1] = h.D1 * d * chi_r; sp.out_sb[2] = 1;
      sp.K = (int)(h.D * d); sp.N = (int)(h.D1 * d);
      sp.k_lo = 1; sp.n_lo = 1;
      sp.in = T1; sp.W = W1.data; sp.out = T2;
      int k = 0;
      for (int64_t w = 0; w < h.D; w++)
        for (int64_t s = 0; s < d; s++, k++) {
          sp.in_koff[k] = w * chi_lo * d * d * chi_r + s * d * chi_r;
          sp.w_koff[k] = (int32_t)(w * h.D1 * d * d + s * d);
        }
      int n = 0;
      for (int64_t v = 0; v < h.D1; v++)
        for (int64_t p = 0; p < d; p++, n++) {
          sp.out_noff[n] = v * d * chi_r + p * chi_r;
          sp.w_noff[n] = (int32_t)(v * d * d + p);
        }
      { tci_status_t _r = run_skinny(ctx, sp); if (_r) return _r; }
    }
    // ---- T3[b,p,q,c,x] = sum_{v,t} T2[b,t,v,p,c] W2[v,x,t,q] (T1 is dead) ----
    T3 = ws + lay.off_x;
    {
      SkinnyProblem sp{};
      sp.dtype = dt;
      sp.nb[0] = chi_lo; sp.nb[1] = d; sp.nb[2] = chi_r;
      sp.in_sb[0] = d * h.D1 * d * chi_r; sp.in_sb[1] = chi_r; sp.in_sb[2] = 1;
      sp.out_sb[0] = d * d * chi_r * h.D2; sp.out_sb[1] = d * chi_r * h.D2; sp.out_sb[2] = h.D2;
      sp.K = (int)(h.D1 * d); sp.N = (int)(d * h.D2);
      sp.k_lo = 1; sp.n_lo = (int)h.D2;
      sp.in = T2; sp.W = W2.data; sp.out = T3;
      int k = 0;
      for (int64_t v = 0; v < h.D1; v++)
        for (int64_t t = 0; t < d; t++, k++) {
          sp.in_koff[k] = v * d * chi_r + t * h.D1 * d * chi_r;
          sp.w_koff[k] = (int32_t)(v * h.D2 * d * d + t * d);
        }
      int n = 0;
      for (int64_t q = 0; q < d; q++)
        for (int64_t x = 0; x < h.D2; x++, n++) {
          sp.out_noff[n] = q * chi_r * h.D2 + x;
          sp.w_noff[n] = (int32_t)(x * d * d + q);
        }
      { tci_status_t _r = run_skinny(ctx, sp); if (_r) return _r; }
    }
  }
  // ---- GEMM4: out[b,p,q,e] = sum_{c,x} T3[b,p,q,c,x] R[c,x,e] ----
  if (stage) TCI_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, stage->ev_R, 0));
  {
    GemmProblem g{};
    g.dtype = dt;
    g.M = chi_lo * d * d; g.K = chi_r * h.D2; g.N = h.chi_ro;
    g.A = T3; g.a_sm = g.K; g.a_sk = 1;
    g.B = R.data; g.b_sk = g.N; g.b_sn = 1;
    g.C = out.data; g.c_sm = g.N;
    set_zalgo(g);
    if (g.N == 1) { g.b_sk = 1; }
    if (stage && g.zalgo == kZOzaki) {
      // the Ozaki GEMM finishes rows chunk by chunk: stream them out
      g.rows_done = stage_rows_out;
      g.rows_user = stage;
      g.max_chunk_rows = stage->chunk_rows;
      { tci_status_t _r = run_gemm(ctx, g); if (_r) return _r; }
      TCI_CUDA_CHECK(stage->err);
    } else if (stage) {
      // DMMA path: row-chunked GEMMs, each chunk copied out behind the next
      const int64_t M = g.M, ch = std::max<int64_t>(1, stage->chunk_rows);
      for (int64_t m0 = 0; m0 < M; m0 += ch) {
        GemmProblem gc = g;
        gc.M = std::min(ch, M - m0);
        gc.A = static_cast<const char *>(g.A) + m0 * g.a_sm * dtype_size(dt);
        gc.C = static_cast<char *>(g.C) + m0 * g.c_sm * dtype_size(dt);
        if (gc.zalgo == kZOzaki && !ozaki_worthwhile(gc.M, gc.N, gc.K, gc.dtype)) gc.zalgo = kZ3M;
        { tci_status_t _r = run_gemm(ctx, gc); if (_r) return _r; }
        stage_rows_out(stage, m0, gc.M);
        TCI_CUDA_CHECK(stage->err);
      }
    } else {
      // peer-memory all-gather fused into the Ozaki CRT epilogue: each
      // finished element also goes to every peer's copy of this slab
      if (gather && dt == TCI_C128 && g.zalgo == kZOzaki && g.splitk <= 1 && !gemm_thin_applies(g)) {
        g.npeer = gather->npeer;
        for (int p = 0; p < gather->npeer; p++) g.peer_C[p] = gather->peer_out[p];
        gather->fused = true;
      }
      tci_status_t _r = run_gemm(ctx, g);
      if (_r) return _r;
    }
  }
  return TCI_OK;
}

// ---------------------------------------------------------------------------
// TEBD theta = (A.B).U (R16)
// ---------------------------------------------------------------------------
tci_status_t tebd_exec(tci_ctx_s *ctx, const View &A, const char *la, const View &B, const char *lb,
                       const View &U, const char *lu, const View &T, const char *lt, size_t *ws_query) {
  if (ws_query) *ws_query = 0;
  const tci_dtype_t dt = A.dtype;
  if (B.dtype != dt || U.dtype != dt || T.dtype != dt)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "tebd: all operands must share one dtype");
  if (dt != TCI_R64 && dt != TCI_C128) TCI_FAIL(TCI_ERR_UNSUPPORTED, "tebd: dtype must be r64 or c128");
  auto len = [](const char *s) { return s ? (int)strlen(s) : -1; };
  if (len(la) != A.order || len(lb) != B.order || len(lu) != U.order || len(lt) != T.order)
    TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "tebd: label string length != tensor order");
  if (A.order != 3 || B.order != 3 || U.order != 4 || T.order != 4)
    TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "tebd: orders must be A 3, B 3, U 4, theta 4");
  // roles: bond = label shared by A and B; s = A label in U; a = other A label
  auto in = [](const char *s, char c) { return strchr(s, c) != nullptr; };
  char bond = 0, s = 0, a = 0, t = 0, c = 0;
  for (int i = 0; i < 3; i++) {
    if (in(lb, la[i])) { if (bond) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "tebd: A and B share > 1 label"); bond = la[i]; }
  }
  if (!bond) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "tebd: A and B share no bond label");
  for (int i = 0; i < 3; i++) {
    if (la[i] != bond) {
      if (in(lu, la[i])) s = la[i]; else a = la[i];
    }
    if (lb[i] != bond) {
      if (in(lu, lb[i])) t = lb[i]; else c = lb[i];
    }
  }
  if (!s || !a || !t || !c) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "tebd: cannot identify physical/bond legs");
  // U = (p,q,s,t) in lu: p,q are the U labels that are not s,t
  char pq[2];
  int npq = 0;
  for (int i = 0; i < 4; i++)
    if (lu[i] != s && lu[i] != t) { if (npq == 2) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "tebd: bad gate labels"); pq[npq++] = lu[i]; }
  if (npq != 2 || in(la, pq[0]) || in(la, pq[1]) || in(lb, pq[0]) || in(lb, pq[1]))
    TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "tebd: gate out legs must be new labels");
  // full label validation of both stages through contract_shape
  int32_t ila[3], ilb[3], ilu[4], ilt[4], iab[4];
  for (int i = 0; i < 3; i++) { ila[i] = (unsigned char)la[i]; ilb[i] = (unsigned char)lb[i]; }
  for (int i = 0; i < 4; i++) { ilu[i] = (unsigned char)lu[i]; ilt[i] = (unsigned char)lt[i]; }
  // AB label order: A's free legs in A order, then B's free legs in B order
  int nab = 0;
  for (int i = 0; i < 3; i++) if (la[i] != bond) iab[nab++] = (unsigned char)la[i];
  for (int i = 0; i < 3; i++) if (lb[i] != bond) iab[nab++] = (unsigned char)lb[i];
  int64_t sab[4], sth[4];
  tci_status_t st = contract_shape(3, A.shape, ila, 3, B.shape, ilb, 4, iab, sab);
  if (st) return st;
  st = contract_shape(4, sab, iab, 4, U.shape, ilu, 4, ilt, sth);
  if (st) return st;
  for (int k = 0; k < 4; k++)
    if (sth[k] != T.shape[k]) TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "tebd: theta shape mismatch");
  // ---- fused path: the gate applied in the GEMM epilogue (d = 2, f64) ----
  {
    auto stride_of = [](const int32_t *l, const int64_t *shape, int n, char x) -> int64_t {
      int64_t st = 1;
      for (int k = n - 1; k >= 0; k--) {
        if (l[k] == (unsigned char)x) return st;
        st *= shape[k];
      }
      return -1;
    };
    TebdProblem tp{};
    tp.d = U.shape[0];
    tp.chi_a = A.shape[strchr(la, a) - la];
    tp.chi_b = A.shape[strchr(la, bond) - la];
    tp.chi_c = B.shape[strchr(lb, c) - lb];
    tp.A = static_cast<const double *>(A.data);
    tp.a_a = stride_of(ila, A.shape, 3, a); tp.a_s = stride_of(ila, A.shape, 3, s); tp.a_b = stride_of(ila, A.shape, 3, bond);
    tp.B = static_cast<const double *>(B.data);
    tp.b_b = stride_of(ilb, B.shape, 3, bond); tp.b_t = stride_of(ilb, B.shape, 3, t); tp.b_c = stride_of(ilb, B.shape, 3, c);
    tp.U = static_cast<const double *>(U.data);
    tp.u_p = stride_of(ilu, U.shape, 4, pq[0]); tp.u_q = stride_of(ilu, U.shape, 4, pq[1]);
    tp.u_s = stride_of(ilu, U.shape, 4, s); tp.u_t = stride_of(ilu, U.shape, 4, t);
    tp.T = static_cast<double *>(T.data);
    tp.t_a = stride_of(ilt, T.shape, 4, a); tp.t_p = stride_of(ilt, T.shape, 4, pq[0]);
    tp.t_q = stride_of(ilt, T.shape, 4, pq[1]); tp.t_c = stride_of(ilt, T.shape, 4, c);
    const bool dims_ok = U.shape[0] == 2 && U.shape[1] == 2 && U.shape[2] == 2 && U.shape[3] == 2 &&
                         A.shape[strchr(la, s) - la] == 2 && B.shape[strchr(lb, t) - lb] == 2;
    // (with the Ozaki algorithm selected, A.B runs as a real Ozaki GEMM and the
    // gate as the skinny pass below; the fused epilogue is a DMMA kernel)
    if (dt == TCI_R64 && dims_ok && ctx->zgemm_algo != kZOzaki && tebd_fused_supported(tp))
      return ws_query ? TCI_OK : run_tebd(ctx, tp);
  }
  View AB;
  AB.dtype = dt;
  AB.order = 4;
  for (int k = 0; k < 4; k++) AB.shape[k] = sab[k];
  const size_t es = dtype_size(dt);
  const size_t ab_bytes = align_up(AB.bytes());
  size_t need_c = 0;
  AB.data = nullptr;
  st = contract_exec(ctx, A, ila, B, ilb, AB, iab, true, &need_c, nullptr, 0);
  if (st) return st;
  // skinny gate pass: batch (a, c), K = (s, t), N = (p, q)
  auto pos = [](const int32_t *l, int n, char x) {
    for (int i = 0; i < n; i++) if (l[i] == (unsigned char)x) return i;
    return -1;
  };
  int64_t abst[4], ust[4], tst[4];
  {
    int64_t v = 1;
    for (int k = 3; k >= 0; k--) { abst[k] = v; v *= sab[k]; }
    v = 1;
    for (int k = 3; k >= 0; k--) { ust[k] = v; v *= U.shape[k]; }
    v = 1;
    for (int k = 3; k >= 0; k--) { tst[k] = v; v *= T.shape[k]; }
  }
  const int64_t ds = sab[pos(iab, 4, s)], dtt = sab[pos(iab, 4, t)];
  const int64_t dp = U.shape[pos(ilu, 4, pq[0])], dq = U.shape[pos(ilu, 4, pq[1])];
  if (ds * dtt > kSkinnyMaxK || dp * dq > kSkinnyMaxN || skinny_smem_bytes((int)(ds * dtt), (int)(dp * dq), es) > 200 * 1024)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "tebd: physical dimension too large for the gate kernel");
  if (ws_query) {
    *ws_query = ab_bytes + need_c;
    return TCI_OK;
  }
  if (ab_bytes + need_c > ctx->ws_bytes || !ctx->ws)
    TCI_FAIL(TCI_ERR_WORKSPACE, "tebd needs %zu bytes of workspace, %zu attached", ab_bytes + need_c,
             ctx->ws_bytes);
  char *ws = static_cast<char *>(ctx->ws);
  AB.data = ws;
  st = contract_exec(ctx, A, ila, B, ilb, AB, iab, false, &need_c, ws + ab_bytes, ctx->ws_bytes - ab_bytes);
  if (st) return st;
  SkinnyProblem sp{};
  sp.dtype = dt;
  // batch legs: b1 = a, b2 = c (c is the bond leg of B: usually fastest)
  sp.nb[0] = 1; sp.nb[1] = sab[pos(iab, 4, a)]; sp.nb[2] = sab[pos(iab, 4, c)];
  sp.in_sb[0] = 0; sp.in_sb[1] = abst[pos(iab, 4, a)]; sp.in_sb[2] = abst[pos(iab, 4, c)];
  sp.out_sb[0] = 0; sp.out_sb[1] = tst[pos(ilt, 4, a)]; sp.out_sb[2] = tst[pos(ilt, 4, c)];
  sp.K = (int)(ds * dtt); sp.N = (int)(dp * dq);
  sp.k_lo = 1; sp.n_lo = 1;
  sp.in = AB.data; sp.W = U.data; sp.out = T.data;
  int k = 0;
  for (int64_t is = 0; is < ds; is++)
    for (int64_t it = 0; it < dtt; it++, k++) {
      sp.in_koff[k] = is * abst[pos(iab, 4, s)] + it * abst[pos(iab, 4, t)];
      sp.w_koff[k] = (int32_t)(is * ust[pos(ilu, 4, s)] + it * ust[pos(ilu, 4, t)]);
    }
  int n = 0;
  for (int64_t ip = 0; ip < dp; ip++)
    for (int64_t iq = 0; iq < dq; iq++, n++) {
      sp.out_noff[n] = ip * tst[pos(ilt, 4, pq[0])] + iq * tst[pos(ilt, 4, pq[1])];
      sp.w_noff[n] = (int32_t)(ip * ust[pos(ilu, 4, pq[0])] + iq * ust[pos(ilu, 4, pq[1])]);
    }
  { tci_status_t _r = run_skinny(ctx, sp); if (_r) return _r; }
  return TCI_OK;
}

}  // namespace tci

// exported diagnostic (include/tci_b200.h): the planner's tree and MAC count
extern "C" int tci_heff_plan_tree(int64_t chi_l, int64_t chi_lo, int64_t chi_r, int64_t chi_ro,
                                  int64_t d, int64_t D, int64_t D1, int64_t D2, char *buf, int n,
                                  double *macs) {
  using namespace tci;
  const int64_t dims[NLAB] = {chi_l, D, chi_lo, d, d, chi_r, D1, d, D2, d, chi_ro};
  std::vector<Node> nd = plan_heff_tree(dims);
  const std::string s = tree_str(nd, 31);
  if (buf && n > 0) snprintf(buf, (size_t)n, "%s", s.c_str());
  if (macs) *macs = nd[31].cost;
  return is_standard_tree(nd) ? 1 : 0;
}
