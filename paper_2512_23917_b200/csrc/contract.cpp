// contract.cpp -- label analysis, leg fusion, GEMM mapping and execution of
// tci_contract.
//
// Semantics (Eq. (3)): labels in both alpha
// and beta but not in gamma are summed; gamma orders the free bonds of c.
// Lowering: matricize A to [I,S], B to [S,J], one GEMM, refold
// to gamma -- but the two permutes and the refold are only materialised when
// the legs do not already FUSE into strided matrices:
//   * extent-1 legs are dropped (they do not move any element);
//   * for each of the 8 choices of (I order in {gamma, A}, J order in
//     {gamma, B}, S order in {A, B}) the planner checks whether A is
//     [I,S] or [S,I], B is [S,J] or [J,S] and gamma is [I,J] or [J,I] as
//     contiguous leg blocks; an operand that fits is read in place by the GEMM
//     loaders (either major-ness), one that does not is permuted into scratch;
//     the choice minimising permuted bytes wins (ties: fixed enumeration order);
//   * gamma == [J,I] is handled by computing C^T = B^T A^T (operand swap).
// The plan depends only on dtype, shapes, the label STRUCTURE (labels are
// canonicalised by first appearance) and aliasing, never on label values, so
// relabelling is bitwise invariant (R23). Plans are cached per
// context under that key.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "runtime.h"

namespace tci {

// TCI_CONTRACT_NO_SKINNY=1 disables the skinny route (A/B measurements)
static bool skinny_route_disabled() {
  static const bool off = [] {
    const char *e = getenv("TCI_CONTRACT_NO_SKINNY");
    return e && *e == '1';
  }();
  return off;
}

static int find_label(int n, const int32_t *l, int32_t x) {
  for (int i = 0; i < n; i++)
    if (l[i] == x) return i;
  return -1;
}

tci_status_t contract_shape(int na, const int64_t *sa, const int32_t *la, int nb, const int64_t *sb,
                            const int32_t *lb, int nc, const int32_t *lc, int64_t *sc) {
  if (na < 0 || nb < 0 || nc < 0) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "negative order");
  if (na > kMaxOrder || nb > kMaxOrder || nc > kMaxOrder)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "order > %d", kMaxOrder);
  for (int i = 0; i < na; i++)
    if (sa[i] < 1) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "a: dimension %d < 1", i);
  for (int i = 0; i < nb; i++)
    if (sb[i] < 1) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "b: dimension %d < 1", i);
  for (int i = 0; i < na; i++)
    if (find_label(i, la, la[i]) >= 0) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "label repeated in a (P:1955)");
  for (int i = 0; i < nb; i++)
    if (find_label(i, lb, lb[i]) >= 0) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "label repeated in b (P:1955)");
  for (int i = 0; i < nc; i++)
    if (find_label(i, lc, lc[i]) >= 0) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "label repeated in c");
  for (int i = 0; i < na; i++) {
    const bool inb = find_label(nb, lb, la[i]) >= 0, inc = find_label(nc, lc, la[i]) >= 0;
    if (inb && inc) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "label in a, b and c (reading R3)");
    if (!inb && !inc) TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "label only in a and not in c (reading R4)");
  }
  for (int i = 0; i < nb; i++) {
    if (find_label(na, la, lb[i]) < 0 && find_label(nc, lc, lb[i]) < 0)
      TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "label only in b and not in c (reading R4)");
  }
  for (int i = 0; i < nc; i++)
    if (find_label(na, la, lc[i]) < 0 && find_label(nb, lb, lc[i]) < 0)
      TCI_FAIL(TCI_ERR_LABEL_CONFLICT, "output label absent from the inputs (reading R5)");
  for (int i = 0; i < na; i++) {
    const int j = find_label(nb, lb, la[i]);
    if (j >= 0 && sa[i] != sb[j])
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "dims of a shared label differ: %lld vs %lld (P:1950)",
               (long long)sa[i], (long long)sb[j]);
  }
  for (int i = 0; i < nc; i++) {
    const int ia = find_label(na, la, lc[i]);
    sc[i] = ia >= 0 ? sa[ia] : sb[find_label(nb, lb, lc[i])];
  }
  return TCI_OK;
}

namespace {

// one leg after dropping extent-1 legs: canonical label id, extent, stride
struct Leg {
  int id;
  int64_t dim, stride;
};

struct Operand {
  int n = 0;
  Leg leg[kMaxOrder];
};

// Target leg order of an operand that must be permuted for the GEMM: [F, S]
// or [S, F] (F its free legs, S the contracted ones), whichever keeps the
// operand's fastest leg fastest -- the GEMM loaders take either major-ness.
static std::vector<int> permute_target(const Operand &o, const std::vector<int> &F, const std::vector<int> &S,
                                       const std::vector<char> &inF) {
  std::vector<int> t;
  const bool fast_free = o.n > 0 && inF[o.leg[o.n - 1].id];
  const std::vector<int> &first = fast_free ? S : F, &second = fast_free ? F : S;
  t.insert(t.end(), first.begin(), first.end());
  t.insert(t.end(), second.begin(), second.end());
  return t;
}
static bool keeps_fastest(const Operand &o, const std::vector<int> &target) {
  return o.n == 0 || target.empty() || target.back() == o.leg[o.n - 1].id;
}

Operand reduce(int order, const int64_t *shape, const int *ids) {
  Operand o;
  int64_t st = 1;
  int64_t strides[kMaxOrder];
  for (int k = order - 1; k >= 0; k--) { strides[k] = st; st *= shape[k]; }
  for (int k = 0; k < order; k++)
    if (shape[k] > 1) o.leg[o.n++] = Leg{ids[k], shape[k], strides[k]};
  return o;
}

// sequence of ids of an operand's legs restricted to `set`
std::vector<int> seq_of(const Operand &o, const std::vector<char> &set) {
  std::vector<int> s;
  for (int k = 0; k < o.n; k++)
    if (set[o.leg[k].id]) s.push_back(o.leg[k].id);
  return s;
}

std::vector<int> ids_of(const Operand &o) {
  std::vector<int> s;
  for (int k = 0; k < o.n; k++) s.push_back(o.leg[k].id);
  return s;
}

std::vector<int> cat(const std::vector<int> &x, const std::vector<int> &y) {
  std::vector<int> r(x);
  r.insert(r.end(), y.begin(), y.end());
  return r;
}

// 0: not blocked; 1: [X,Y]; 2: [Y,X]
int blocks(const std::vector<int> &legs, const std::vector<int> &X, const std::vector<int> &Y) {
  if (legs == cat(X, Y)) return 1;
  if (legs == cat(Y, X)) return 2;
  return 0;
}

int64_t extent(const std::vector<int> &ids, const int64_t *dim_of) {
  int64_t e = 1;
  for (int id : ids) e *= dim_of[id];
  return e;
}

}  // namespace

// Plan decision vector layout (cached): [order choice, formA, formB, formC]
//   formX: 0 = permute into scratch, 1 / 2 = blocks as documented above
tci_status_t contract_exec(tci_ctx_s *ctx, const View &a, const int32_t *la, const View &b,
                           const int32_t *lb, const View &c, const int32_t *lc, bool dry_run,
                           size_t *ws_needed, void *ws, size_t ws_bytes) {
  if (a.dtype != b.dtype || a.dtype != c.dtype)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "operands must share one dtype (one TenT per call, P:1918)");
  int64_t sc[kMaxOrder];
  tci_status_t st = contract_shape(a.order, a.shape, la, b.order, b.shape, lb, c.order, lc, sc);
  if (st != TCI_OK) return st;
  for (int k = 0; k < c.order; k++)
    if (sc[k] != c.shape[k])
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "c.shape[%d] = %lld, contraction gives %lld", k,
               (long long)c.shape[k], (long long)sc[k]);

  // canonical label ids by first appearance (a, then b, then c)
  int ida[kMaxOrder], idb[kMaxOrder], idc[kMaxOrder];
  int32_t uniq[3 * kMaxOrder];
  int nu = 0;
  auto canon = [&](int32_t l) {
    for (int i = 0; i < nu; i++)
      if (uniq[i] == l) return i;
    uniq[nu] = l;
    return nu++;
  };
  for (int k = 0; k < a.order; k++) ida[k] = canon(la[k]);
  for (int k = 0; k < b.order; k++) idb[k] = canon(lb[k]);
  for (int k = 0; k < c.order; k++) idc[k] = canon(lc[k]);
  int64_t dim_of[3 * kMaxOrder];
  for (int k = 0; k < a.order; k++) dim_of[ida[k]] = a.shape[k];
  for (int k = 0; k < b.order; k++) dim_of[idb[k]] = b.shape[k];

  const Operand A = reduce(a.order, a.shape, ida);
  const Operand B = reduce(b.order, b.shape, idb);
  const Operand C = reduce(c.order, c.shape, idc);

  std::vector<char> inI(nu, 0), inJ(nu, 0), inS(nu, 0);
  for (int k = 0; k < A.n; k++) {
    bool in_b = false;
    for (int j = 0; j < B.n; j++) in_b |= B.leg[j].id == A.leg[k].id;
    (in_b ? inS : inI)[A.leg[k].id] = 1;
  }
  for (int j = 0; j < B.n; j++)
    if (!inS[B.leg[j].id]) inJ[B.leg[j].id] = 1;

  const std::vector<int> Ig = seq_of(C, inI), Ia = seq_of(A, inI);
  const std::vector<int> Jg = seq_of(C, inJ), Jb = seq_of(B, inJ);
  const std::vector<int> Sa = seq_of(A, inS), Sb = seq_of(B, inS);
  const std::vector<int> legsA = ids_of(A), legsB = ids_of(B), legsC = ids_of(C);

  // aliasing: output range overlapping an input range
  auto overlap = [](const void *p, size_t np, const void *q, size_t nq) {
    const char *x = static_cast<const char *>(p), *y = static_cast<const char *>(q);
    return np && nq && x < y + nq && y < x + np;
  };
  const bool alias = overlap(c.data, c.bytes(), a.data, a.bytes()) ||
                     overlap(c.data, c.bytes(), b.data, b.bytes());

  // ---- skinny route (8(a5), 8(a10)): one small operand W (contracted
  // extent K <= 64, free extent <= 128) against a large one X whose free legs
  // form at most three (fused) batch groups: out[b, n] = sum_k X[b, k] W(k, n)
  // streamed once through the skinny kernel, written in gamma order directly
  // (no GEMM tile, no permute). f64 / c128, no aliasing.
  if (!alias && (a.dtype == TCI_R64 || a.dtype == TCI_C128) && !skinny_route_disabled()) {
    int64_t KS = 1;
    for (int k = 0; k < A.n; k++)
      if (inS[A.leg[k].id]) KS *= A.leg[k].dim;
    auto sin = [](const Operand &o, int id) {
      for (int k = 0; k < o.n; k++)
        if (o.leg[k].id == id) return o.leg[k].stride;
      return (int64_t)0;
    };
    for (int side = 0; side < 2 && KS <= 64; side++) {
      const Operand &X = side == 0 ? A : B, &Wo = side == 0 ? B : A;
      const int64_t nW = side == 0 ? b.size() : a.size(), nX = side == 0 ? a.size() : b.size();
      if (nW * 16 > nX || nW > 64 * 128) continue;
      const std::vector<char> &freeW = side == 0 ? inJ : inI;
      const std::vector<char> &freeX = side == 0 ? inI : inJ;
      int64_t NW = 1;
      for (int k = 0; k < Wo.n; k++)
        if (freeW[Wo.leg[k].id]) NW *= Wo.leg[k].dim;
      if (NW > kSkinnyMaxN || KS > kSkinnyMaxK) continue;
      // batch groups: X's free legs in X order (slowest first), fused when
      // adjacent with matching strides in both X and C
      int64_t gext[kMaxOrder], gin[kMaxOrder], gout[kMaxOrder];
      int ng = 0;
      for (int k = 0; k < X.n; k++) {
        const int id = X.leg[k].id;
        if (!freeX[id]) continue;
        const int64_t e = X.leg[k].dim, si = X.leg[k].stride, so = sin(C, id);
        if (ng > 0 && gin[ng - 1] == si * e && gout[ng - 1] == so * e) {
          gext[ng - 1] *= e;
          gin[ng - 1] = si;
          gout[ng - 1] = so;
        } else {
          gext[ng] = e;
          gin[ng] = si;
          gout[ng] = so;
          ng++;
        }
      }
      if (ng > 3) continue;
      SkinnyProblem sp{};
      sp.dtype = a.dtype;
      for (int g = 0; g < 3; g++) {
        const int src = g - (3 - ng);
        sp.nb[g] = src >= 0 ? gext[src] : 1;
        sp.in_sb[g] = src >= 0 ? gin[src] : 0;
        sp.out_sb[g] = src >= 0 ? gout[src] : 0;
      }
      sp.K = (int)KS;
      sp.N = (int)NW;
      // k enumerates the contracted legs in X order; n the free legs of W
      // ordered by decreasing C stride (the fastest C leg innermost)
      std::vector<int> kl, nl;
      for (int k = 0; k < X.n; k++)
        if (inS[X.leg[k].id]) kl.push_back(X.leg[k].id);
      for (int k = 0; k < Wo.n; k++)
        if (freeW[Wo.leg[k].id]) nl.push_back(Wo.leg[k].id);
      std::stable_sort(nl.begin(), nl.end(), [&](int x, int y) { return sin(C, x) > sin(C, y); });
      auto fill = [&](const std::vector<int> &legs, const Operand &o1, int64_t *off1, const Operand &o2,
                      int32_t *off2, int64_t total) {
        for (int64_t i = 0; i < total; i++) {
          int64_t r = i, a1 = 0, a2 = 0;
          for (int q = (int)legs.size() - 1; q >= 0; q--) {
            const int64_t e = dim_of[legs[q]], c_ = r % e;
            r /= e;
            a1 += c_ * sin(o1, legs[q]);
            a2 += c_ * sin(o2, legs[q]);
          }
          off1[i] = a1;
          off2[i] = (int32_t)a2;
        }
      };
      fill(kl, X, sp.in_koff, Wo, sp.w_koff, KS);
      fill(nl, C, sp.out_noff, Wo, sp.w_noff, NW);
      sp.k_lo = 1;
      sp.n_lo = 1;
      if (!nl.empty() && sin(C, nl.back()) == 1 && sp.out_sb[2] == dim_of[nl.back()]) sp.n_lo = (int)dim_of[nl.back()];
      sp.in = side == 0 ? a.data : b.data;
      sp.W = side == 0 ? b.data : a.data;
      sp.out = c.data;
      *ws_needed = 0;
      if (dry_run) return TCI_OK;
      return run_skinny(ctx, sp);
    }
  }

  // ---- plan choice (cached) ----
  // binary key: dtype, alias, then (extent, canonical id) per leg of a, b, c
  std::string key;
  {
    int64_t buf[2 + 6 * kMaxOrder + 3];
    int nk = 0;
    buf[nk++] = (int64_t)a.dtype;
    buf[nk++] = (int64_t)alias;
    auto put = [&](int n, const int64_t *s, const int *ids) {
      buf[nk++] = n;
      for (int k = 0; k < n; k++) {
        buf[nk++] = s[k];
        buf[nk++] = ids[k];
      }
    };
    put(a.order, a.shape, ida);
    put(b.order, b.shape, idb);
    put(c.order, c.shape, idc);
    key.assign(reinterpret_cast<const char *>(buf), nk * sizeof(int64_t));
  }
  int choice = -1, formA = 0, formB = 0, formC = 0;
  auto it = ctx->plan_cache.find(key);
  if (it != ctx->plan_cache.end()) {
    choice = (int)it->second[0];
    formA = (int)it->second[1];
    formB = (int)it->second[2];
    formC = (int)it->second[3];
    ctx->plan_hits++;
  } else {
    const int64_t nA = a.size(), nB = b.size(), nC = c.size();
    int64_t best = -1;
    for (int ch = 0; ch < 8; ch++) {
      const std::vector<int> &I = (ch & 1) ? Ia : Ig;
      const std::vector<int> &J = (ch & 2) ? Jb : Jg;
      const std::vector<int> &S = (ch & 4) ? Sb : Sa;
      const int fa = blocks(legsA, I, S), fb = blocks(legsB, S, J), fc = blocks(legsC, I, J);
      // a permute that keeps the operand's fastest leg fastest runs as row
      // copies (~5.5 TB/s); one that moves it is a transpose (~2-3 TB/s):
      // those bytes count twice
      const int64_t pa = fa ? 0 : 2 * nA * (keeps_fastest(A, permute_target(A, I, S, inI)) ? 1 : 2);
      const int64_t pb = fb ? 0 : 2 * nB * (keeps_fastest(B, permute_target(B, J, S, inJ)) ? 1 : 2);
      const bool c_keeps = C.n == 0 || (!I.empty() && C.leg[C.n - 1].id == I.back()) ||
                           (!J.empty() && C.leg[C.n - 1].id == J.back());
      const int64_t pc = fc ? 0 : 2 * nC * (c_keeps ? 1 : 2);
      const int64_t cost = pa + pb + pc;
      if (best < 0 || cost < best) {
        best = cost;
        choice = ch;
        formA = fa;
        formB = fb;
        formC = fc;
      }
    }
    ctx->plan_cache[key] = {choice, formA, formB, formC};
    ctx->plan_misses++;
  }
  const std::vector<int> &I = (choice & 1) ? Ia : Ig;
  const std::vector<int> &J = (choice & 2) ? Jb : Jg;
  const std::vector<int> &S = (choice & 4) ? Sb : Sa;
  const int64_t M = extent(I, dim_of), N = extent(J, dim_of), K = extent(S, dim_of);
  const size_t es = dtype_size(a.dtype);

  // the INT8 tensor-core path (Ozaki-II) for this dtype under the context's
  // choice: float64 / complex128 when the GEMM algorithm is Ozaki, float32 /
  // complex64 unless the context keeps them on the FP64 cores (R34)
  const bool oz_dtype = ((a.dtype == TCI_C128 || a.dtype == TCI_R64) && ctx->zgemm_algo == kZOzaki) ||
                        ((a.dtype == TCI_R32 || a.dtype == TCI_C64) && ctx->f32_algo == TCI_F32_OZAKI_INT8);
  // deterministic split-K when the output has too few tiles to fill the 148
  // SMs and K is long: S partial GEMMs over K chunks + an ascending-order sum
  int splitk = 1;
  int64_t k_chunk = 0;
  size_t offP = 0;
  {
    int bm, bn;
    gemm_tile(a.dtype, &bm, &bn);
    // thin GEMMs (gemm_thin.cu: one thread / warp per row of the long side)
    // parallelise over 256-row blocks, not GEMM tiles
    const bool thin = std::min(M, N) <= (dtype_is_complex(a.dtype) ? 16 : 32);
    const int64_t tiles = thin ? (std::max(M, N) + 255) / 256 : ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
    // (not when the GEMM goes to the INT8 tensor cores: its 3n / n residue
    // GEMMs of one launch fill the machine by themselves)
    const bool oz_candidate = oz_dtype && ozaki_worthwhile(M, N, K, a.dtype);
    if (tiles < 2 * 148 && K >= 256 && !oz_candidate) {
      int64_t S = std::min<int64_t>({(4 * 148 + tiles - 1) / tiles, K / 64, 1024});
      if (S >= 2) {
        k_chunk = ((K + S - 1) / S + 15) / 16 * 16;
        S = (K + k_chunk - 1) / k_chunk;
        if (S >= 2) splitk = (int)S;
      }
    }
  }
  // complex128 GEMM algorithm
  int zalgo = ctx->zgemm_algo == kZOzaki ? kZ3M : ctx->zgemm_algo;
  // (float64 too: real Ozaki-II, one residue plane per modulus)
  const bool use_ozaki = oz_dtype && splitk <= 1 && ozaki_worthwhile(M, N, K, a.dtype);
  // gamma-order scatter epilogue (8(a6)): an output that is not a [I,J] /
  // [J,I] block is written in place through row / column offset tables
  // instead of GEMM -> scratch -> permute; the GEMM is oriented so that the
  // fastest gamma leg is on its N side (coalesced runs)
  bool scatter = !formC && !alias && !use_ozaki && C.n > 0;
  bool scat_swap = false;
  if (scatter) {
    scat_swap = inI[C.leg[C.n - 1].id] != 0;
    // contiguous gamma run along the GEMM's N side: the trailing gamma legs
    // that are also the trailing legs of the N-side order; short runs write
    // scattered sectors, so below 128 bytes the GEMM -> scratch -> permute
    // route (leg-group tiles) is the better one
    const std::vector<int> &Nside = scat_swap ? I : J;
    int64_t run = 1;
    int pos = (int)Nside.size() - 1;
    for (int k = C.n - 1; k >= 0 && pos >= 0 && C.leg[k].id == Nside[pos]; k--, pos--) run *= C.leg[k].dim;
    // (a pure output-write kernel, K <= 16, needs whole 128-byte lines; with a
    // real K the GEMM hides partial sectors up to one 32-byte sector per run)
    if (run * (int64_t)es < (K <= 16 ? 128 : 32)) scatter = false;
  }

  // ---- scratch layout ----
  size_t off = 0, offA = 0, offB = 0, offC = 0, offR = 0, offCol = 0;
  if (!formA) { offA = off; off = align_up(off + (size_t)M * K * es); }
  if (!formB) { offB = off; off = align_up(off + (size_t)K * N * es); }
  const bool c_scratch = (!formC && !scatter) || alias;
  if (c_scratch) { offC = off; off = align_up(off + (size_t)M * N * es); }
  if (scatter) {
    offR = off;
    off = align_up(off + (size_t)M * 8);
    offCol = off;
    off = align_up(off + (size_t)N * 8);
  }
  if (splitk > 1) {
    const size_t pes = dtype_is_complex(a.dtype) ? 16 : 8;   // fp64 partials
    offP = off;
    off = align_up(off + (size_t)splitk * M * N * pes);
  }
  size_t offZ = 0, ozb = 0;
  if (use_ozaki) {
    zalgo = kZOzaki;
    ozb = ozaki_workspace_bytes(M, N, K);
    offZ = off;
    off = align_up(off + ozb);
  }
  *ws_needed = off;
  if (dry_run) return TCI_OK;
  if (off > ws_bytes || (off && !ws))
    TCI_FAIL(TCI_ERR_WORKSPACE, "contract needs %zu bytes of workspace, %zu attached", off, ws_bytes);
  char *wsb = static_cast<char *>(ws);

  auto stride_in = [](const Operand &o, int id) {
    for (int k = 0; k < o.n; k++)
      if (o.leg[k].id == id) return o.leg[k].stride;
    return (int64_t)0;
  };
  // permute the legs of operand `o` (data `src`) into order `ord` at `dst`
  auto permute_into = [&](const Operand &o, const void *src, const std::vector<int> &ord,
                          void *dst) -> tci_status_t {
    PermuteProblem pp{};
    pp.esize = es;
    pp.in = src;
    pp.out = dst;
    pp.total = 1;
    // fuse adjacent out legs that are adjacent in the input too
    int n = 0;
    for (size_t k = 0; k < ord.size(); k++) {
      const int64_t d = dim_of[ord[k]], s = stride_in(o, ord[k]);
      if (n > 0 && pp.in_stride_for_out[n - 1] == s * d) {
        pp.shape_out[n - 1] *= d;
        pp.in_stride_for_out[n - 1] = s;
      } else {
        pp.shape_out[n] = d;
        pp.in_stride_for_out[n] = s;
        n++;
      }
      pp.total *= d;
    }
    pp.n = n;
    { tci_status_t _r = run_permute(ctx, pp); if (_r) return _r; }
    return TCI_OK;
  };

  // ---- operand A as a strided [M x K] matrix ----
  GemmProblem g{};
  g.dtype = a.dtype;
  g.M = M; g.N = N; g.K = K;
  const void *Ap = a.data;
  int fa = formA;
  if (!formA) {
    const std::vector<int> tA = permute_target(A, I, S, inI);
    st = permute_into(A, a.data, tA, wsb + offA);
    if (st != TCI_OK) return st;
    Ap = wsb + offA;
    fa = (!S.empty() && tA.back() == S.back()) || I.empty() ? 1 : 2;   // [I, S] or [S, I]
  }
  if (fa == 1) { g.a_sm = K; g.a_sk = 1; }   // [I, S]
  else { g.a_sm = 1; g.a_sk = M; }           // [S, I]
  const void *Bp = b.data;
  int fb = formB;
  if (!formB) {
    const std::vector<int> tB = permute_target(B, J, S, inJ);   // [J, S] or [S, J]
    st = permute_into(B, b.data, tB, wsb + offB);
    if (st != TCI_OK) return st;
    Bp = wsb + offB;
    fb = (!J.empty() && tB.back() == J.back()) || S.empty() ? 1 : 2;   // [S, J] or [J, S]
  }
  if (fb == 1) { g.b_sk = N; g.b_sn = 1; }   // [S, J]
  else { g.b_sk = 1; g.b_sn = K; }           // [J, S]
  g.A = Ap;
  g.B = Bp;
  // canonicalise degenerate extents (gemm_dmma.cu contract: a_sk == 1 picks
  // the K-contiguous loader, else a_sm must be 1)
  auto canon_a = [](int64_t M_, int64_t K_, int64_t &sm, int64_t &sk) {
    if (K_ == 1) { if (sm == 1 && M_ > 1) sk = 0; else { sk = 1; if (M_ == 1) sm = 1; } }
    else if (M_ == 1 && sk != 1) sm = 1;
  };
  // C layout: formC == 2 means gamma = [J, I] -> swap roles (also for a
  // scatter whose fastest gamma leg is an I leg)
  // (and a GEMM -> scratch -> refold whose fastest gamma leg is an I leg: the
  // scratch then holds [J, I], so the refold keeps that leg fastest)
  const bool c_swap_refold = c_scratch && !alias && !formC && !scatter && C.n > 0 && inI[C.leg[C.n - 1].id];
  const bool swap = (((formC == 2) || (scatter && scat_swap)) && !alias) || c_swap_refold;
  void *Cp = c_scratch ? (void *)(wsb + offC) : c.data;
  int64_t *rowt = nullptr, *colt = nullptr;
  if (scatter) {
    // gamma offsets of the I legs (rows) and J legs (columns), slowest first:
    // both tables in one launch
    int64_t exi[kMaxOrder], sti[kMaxOrder], exj[kMaxOrder], stj[kMaxOrder];
    int ni = 0, nj = 0;
    for (int id : I) { exi[ni] = dim_of[id]; sti[ni] = stride_in(C, id); ni++; }
    for (int id : J) { exj[nj] = dim_of[id]; stj[nj] = stride_in(C, id); nj++; }
    int64_t *ti = reinterpret_cast<int64_t *>(wsb + offR), *tj = reinterpret_cast<int64_t *>(wsb + offCol);
    TCI_CUDA_CHECK(launch_offsets2(ti, M, ni, exi, sti, tj, N, nj, exj, stj, ctx->stream, &ctx->launches));
    rowt = swap ? tj : ti;
    colt = swap ? ti : tj;
  }
  if (!swap) {
    g.C = Cp;
    g.c_sm = N;
  } else {
    GemmProblem t = g;
    t.M = N; t.N = M;
    t.A = Bp; t.a_sm = g.b_sn; t.a_sk = g.b_sk;
    t.B = Ap; t.b_sk = g.a_sk; t.b_sn = g.a_sm;
    t.C = Cp; t.c_sm = M;
    g = t;
  }
  canon_a(g.M, g.K, g.a_sm, g.a_sk);
  // B(k,n): the same rule with (N, K)
  canon_a(g.N, g.K, g.b_sn, g.b_sk);
  g.c_row = rowt;
  g.c_col = colt;
  g.zalgo = zalgo;
  if (zalgo == kZOzaki) {
    g.oz_ws = wsb + offZ;
    g.oz_ws_bytes = ozb;
  }
  if (splitk > 1) {
    g.splitk = splitk;
    g.k_chunk = k_chunk;
    g.partial = wsb + offP;
  }
  { tci_status_t _r = run_gemm(ctx, g); if (_r) return _r; }

  // ---- refold into gamma order (or copy out of scratch when aliased) ----
  if (c_scratch) {
    if (formC == 1 || (formC == 2 && swap)) {
      TCI_CUDA_CHECK(launch_copy(c.data, Cp, c.bytes(), ctx->stream, &ctx->launches));
    } else {
      // scratch holds [I, J], or [J, I] after the operand swap
      Operand Ct;
      Ct.n = 0;
      const std::vector<int> IJ = swap ? cat(J, I) : cat(I, J);
      int64_t s = 1;
      int64_t strides[2 * kMaxOrder];
      for (int k = (int)IJ.size() - 1; k >= 0; k--) { strides[k] = s; s *= dim_of[IJ[k]]; }
      for (size_t k = 0; k < IJ.size(); k++) Ct.leg[Ct.n++] = Leg{IJ[k], dim_of[IJ[k]], strides[k]};
      st = permute_into(Ct, Cp, legsC, c.data);
      if (st != TCI_OK) return st;
    }
  }
  return TCI_OK;
}

tci_status_t permute_exec(tci_ctx_s *ctx, const View &in, const int32_t *perm, void *out_data) {
  const size_t es = dtype_size(in.dtype);
  int64_t strides[kMaxOrder];
  int64_t s = 1;
  for (int k = in.order - 1; k >= 0; k--) { strides[k] = s; s *= in.shape[k]; }
  PermuteProblem pp{};
  pp.esize = es;
  pp.in = in.data;
  pp.out = out_data;
  pp.total = in.size();
  int n = 0;
  for (int k = 0; k < in.order; k++) {
    const int64_t d = in.shape[perm[k]], st = strides[perm[k]];
    if (d == 1) continue;
    if (n > 0 && pp.in_stride_for_out[n - 1] == st * d) {
      pp.shape_out[n - 1] *= d;
      pp.in_stride_for_out[n - 1] = st;
    } else {
      pp.shape_out[n] = d;
      pp.in_stride_for_out[n] = st;
      n++;
    }
  }
  pp.n = n;
  { tci_status_t _r = run_permute(ctx, pp); if (_r) return _r; }
  return TCI_OK;
}

}  // namespace tci
