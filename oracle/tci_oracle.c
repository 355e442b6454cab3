/*
 * tci_oracle.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library. The product path
 * (paper_2512_23917_b200/) never links, imports or executes it, and shares
 * no code, header, table or constant with it.
 *
 * What it computes: TCI `contract` and `transpose` exactly as the paper
 * defines them, in double precision, by plain loops:
 *
 *   - transpose, Eq. (1), PAPER.md:167-174 (section II.B "Transpose"):
 *         B_{i_pi(0) i_pi(1) ... i_pi(n-1)} = A_{i_0 i_1 ... i_{n-1}}
 *     i.e. output bond k is input bond pi(k): shape_out[k] = shape_in[pi[k]].
 *     API: PAPER.md:1190-1231 (App. C, tci::transpose).
 *
 *   - contract, Eq. (3), PAPER.md:210-217 (section II.B "Contraction"):
 *         C_{IJ} = sum_S A_{IS} B_{SJ}
 *     with the label rules of PAPER.md:1946-1955 (App. C, tci::contract):
 *     labels in both alpha and beta but not in gamma are summed; gamma gives
 *     the free bonds of c and their order; equal labels must have equal
 *     dimensions; empty gamma gives an order-0 (one element) result; a label
 *     repeated within one operand is prohibited.
 *     It is evaluated the way the paper lowers a tensor linear-algebra
 *     operation (section II.B.2): (i) matricize A to [I,S] and
 *     B to [S,J] with the transpose above, (ii) a plain matrix product with
 *     each element summed over S in ascending row-major order, (iii) refold
 *     [I,J] into gamma order with the transpose above.
 *
 * Layout: row-major, last index fastest (reading R1). Complex
 * values are interleaved (re, im) doubles. The complex product uses the
 * textbook formula (ar*br - ai*bi, ar*bi + ai*br) with separate multiplies
 * and adds; the file is compiled with -ffp-contract=off so no FMA is formed.
 *
 * Parallelism: OpenMP over (row, column-block) pairs of the matricized
 * product only. Each output element is still summed by one thread in
 * ascending S order, so results are bitwise independent of thread count.
 *
 * Status codes mirror DESIGN.md section "Error kinds" (same numbers as the
 * product ABI by specification, but defined here independently).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum {
  OR_OK = 0,
  OR_SHAPE_MISMATCH = 1,
  OR_ORDER_MISMATCH = 2,
  OR_OUT_OF_RANGE = 3,
  OR_LABEL_CONFLICT = 4,
  OR_PARSE = 5,
  OR_UNSUPPORTED = 7,
  OR_INVALID_ARGUMENT = 8,
  OR_NOMEM = 12
};

#define OR_MAX_ORDER 16

/* ------------------------------------------------------------------ */
/* transpose, Eq. (1): out[c_out] = in[c_in] with c_in[perm[k]] = c_out[k] */
/* ------------------------------------------------------------------ */
static int64_t prod(int n, const int64_t *s) {
  int64_t p = 1;
  for (int i = 0; i < n; i++) p *= s[i];
  return p;
}

/* elem = 1 (real double) or 2 (complex, two doubles) */
static void permute_plain(int elem, int n, const int64_t *shape_in,
                          const int32_t *perm, const double *in, double *out,
                          int nthreads) {
  int64_t stride_in[OR_MAX_ORDER], shape_out[OR_MAX_ORDER];
  int64_t total = prod(n, shape_in);
  if (n > 0) stride_in[n - 1] = 1;
  for (int k = n - 2; k >= 0; k--) stride_in[k] = stride_in[k + 1] * shape_in[k + 1];
  for (int k = 0; k < n; k++) shape_out[k] = shape_in[perm[k]];
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
  for (int64_t lin = 0; lin < total; lin++) {
    /* decompose lin into output coordinates (row-major) */
    int64_t rem = lin, off_in = 0;
    for (int k = n - 1; k >= 0; k--) {
      int64_t c = rem % shape_out[k];
      rem /= shape_out[k];
      off_in += c * stride_in[perm[k]]; /* c_in[perm[k]] = c_out[k] */
    }
    for (int e = 0; e < elem; e++) out[lin * elem + e] = in[off_in * elem + e];
  }
  (void)nthreads;
}

int oracle_permute(int is_complex, int n, const int64_t *shape_in,
                   const int32_t *perm, const double *in, double *out,
                   int nthreads) {
  if (n < 0 || n > OR_MAX_ORDER) return OR_UNSUPPORTED;
  int seen[OR_MAX_ORDER] = {0};
  for (int k = 0; k < n; k++) {
    if (shape_in[k] < 1) return OR_OUT_OF_RANGE;
    if (perm[k] < 0 || perm[k] >= n || seen[perm[k]]) return OR_INVALID_ARGUMENT;
    seen[perm[k]] = 1;
  }
  permute_plain(is_complex ? 2 : 1, n, shape_in, perm, in, out, nthreads);
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* contract, Eq. (3) with the rules of PAPER.md:1946-1955               */
/* ------------------------------------------------------------------ */
static int find(int n, const int32_t *l, int32_t x) {
  for (int i = 0; i < n; i++)
    if (l[i] == x) return i;
  return -1;
}

/* Validation, in the documented order. Writes
 * the output shape (gamma order) when successful. */
int oracle_contract_shape(int na, const int64_t *sa, const int32_t *la,
                          int nb, const int64_t *sb, const int32_t *lb,
                          int nc, const int32_t *lc, int64_t *sc) {
  if (na < 0 || nb < 0 || nc < 0) return OR_INVALID_ARGUMENT;
  if (na > OR_MAX_ORDER || nb > OR_MAX_ORDER || nc > OR_MAX_ORDER) return OR_UNSUPPORTED;
  for (int i = 0; i < na; i++) if (sa[i] < 1) return OR_OUT_OF_RANGE;
  for (int i = 0; i < nb; i++) if (sb[i] < 1) return OR_OUT_OF_RANGE;
  /* repeated label within one operand or within gamma */
  for (int i = 0; i < na; i++) if (find(i, la, la[i]) >= 0) return OR_LABEL_CONFLICT;
  for (int i = 0; i < nb; i++) if (find(i, lb, lb[i]) >= 0) return OR_LABEL_CONFLICT;
  for (int i = 0; i < nc; i++) if (find(i, lc, lc[i]) >= 0) return OR_LABEL_CONFLICT;
  /* a label of alpha: in beta (contracted, must not be in gamma) or in gamma */
  for (int i = 0; i < na; i++) {
    int inb = find(nb, lb, la[i]) >= 0, inc = find(nc, lc, la[i]) >= 0;
    if (inb && inc) return OR_LABEL_CONFLICT;   /* reading R3 */
    if (!inb && !inc) return OR_LABEL_CONFLICT; /* reading R4 */
  }
  for (int i = 0; i < nb; i++) {
    int ina = find(na, la, lb[i]) >= 0, inc = find(nc, lc, lb[i]) >= 0;
    if (!ina && !inc) return OR_LABEL_CONFLICT; /* reading R4 */
  }
  for (int i = 0; i < nc; i++) {
    if (find(na, la, lc[i]) < 0 && find(nb, lb, lc[i]) < 0)
      return OR_LABEL_CONFLICT;                 /* reading R5 */
  }
  /* bond dimensions of identical labels must agree */
  for (int i = 0; i < na; i++) {
    int j = find(nb, lb, la[i]);
    if (j >= 0 && sa[i] != sb[j]) return OR_SHAPE_MISMATCH;
  }
  for (int i = 0; i < nc; i++) {
    int ia = find(na, la, lc[i]);
    sc[i] = ia >= 0 ? sa[ia] : sb[find(nb, lb, lc[i])];
  }
  return OR_OK;
}

int oracle_contract(int is_complex,
                    int na, const int64_t *sa, const int32_t *la, const double *A,
                    int nb, const int64_t *sb, const int32_t *lb, const double *B,
                    int nc, const int32_t *lc, double *C, int nthreads) {
  int64_t sc[OR_MAX_ORDER];
  int st = oracle_contract_shape(na, sa, la, nb, sb, lb, nc, lc, sc);
  if (st != OR_OK) return st;
  if (nthreads < 1) nthreads = 1;
  const int elem = is_complex ? 2 : 1;

  /* Bond sets: S = labels of alpha also in beta (alpha
   * order); I = labels of alpha in gamma (alpha order); J = labels of beta
   * in gamma (beta order). */
  int32_t permA[OR_MAX_ORDER], permB[OR_MAX_ORDER], permC[OR_MAX_ORDER];
  int nI = 0, nS = 0, nJ = 0;
  int64_t dimI = 1, dimS = 1, dimJ = 1;
  int32_t labIJ[2 * OR_MAX_ORDER];
  /* A matricized as [I..., S...] */
  for (int i = 0; i < na; i++)
    if (find(nc, lc, la[i]) >= 0) { permA[nI] = i; labIJ[nI] = la[i]; dimI *= sa[i]; nI++; }
  for (int i = 0; i < na; i++)
    if (find(nb, lb, la[i]) >= 0) { permA[nI + nS] = i; dimS *= sa[i]; nS++; }
  /* B matricized as [S..., J...]; S in the same (alpha) order as in A */
  for (int s = 0; s < nS; s++) permB[s] = find(nb, lb, la[permA[nI + s]]);
  for (int j = 0; j < nb; j++)
    if (find(nc, lc, lb[j]) >= 0) { permB[nS + nJ] = j; labIJ[nI + nJ] = lb[j]; dimJ *= sb[j]; nJ++; }

  double *Am = (double *)malloc((size_t)(dimI * dimS * elem) * sizeof(double));
  double *Bm = (double *)malloc((size_t)(dimS * dimJ * elem) * sizeof(double));
  double *Cm = (double *)malloc((size_t)(dimI * dimJ * elem) * sizeof(double));
  if (!Am || !Bm || !Cm) { free(Am); free(Bm); free(Cm); return OR_NOMEM; }

  /* (i) matricize: transposes per Eq. (1) */
  permute_plain(elem, na, sa, permA, A, Am, nthreads);
  permute_plain(elem, nb, sb, permB, B, Bm, nthreads);

  /* (ii) Cm[i,j] = sum_s Am[i,s] * Bm[s,j], s ascending for every element */
  const int64_t JB = 256; /* column block: only splits work between threads */
  const int64_t njb = (dimJ + JB - 1) / JB;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
  for (int64_t task = 0; task < dimI * njb; task++) {
    const int64_t i = task / njb, j0 = (task % njb) * JB;
    const int64_t j1 = j0 + JB < dimJ ? j0 + JB : dimJ;
    double *crow = Cm + i * dimJ * elem;
    for (int64_t j = j0; j < j1; j++)
      for (int e = 0; e < elem; e++) crow[j * elem + e] = 0.0;
    for (int64_t s = 0; s < dimS; s++) {
      const double *brow = Bm + s * dimJ * elem;
      if (!is_complex) {
        const double a = Am[i * dimS + s];
        for (int64_t j = j0; j < j1; j++) {
          double p = a * brow[j];
          crow[j] = crow[j] + p;
        }
      } else {
        const double ar = Am[(i * dimS + s) * 2], ai = Am[(i * dimS + s) * 2 + 1];
        for (int64_t j = j0; j < j1; j++) {
          const double br = brow[2 * j], bi = brow[2 * j + 1];
          double rr = ar * br, ii = ai * bi, ri = ar * bi, ir = ai * br;
          double pr = rr - ii, pi = ri + ir;
          crow[2 * j] = crow[2 * j] + pr;
          crow[2 * j + 1] = crow[2 * j + 1] + pi;
        }
      }
    }
  }

  /* (iii) refold: Cm has bonds [I..., J...] with labels labIJ; gamma order
   * is reached by the transpose with output bond k = Cm bond permC[k]. */
  int64_t sIJ[2 * OR_MAX_ORDER];
  for (int k = 0; k < nI + nJ; k++) {
    int ia = find(na, la, labIJ[k]);
    sIJ[k] = ia >= 0 ? sa[ia] : sb[find(nb, lb, labIJ[k])];
  }
  for (int k = 0; k < nc; k++) permC[k] = find(nI + nJ, labIJ, lc[k]);
  permute_plain(elem, nc, sIJ, permC, Cm, C, nthreads);

  free(Am); free(Bm); free(Cm);
  return OR_OK;
}

/* |A|.|B| contraction: the same loops on element moduli (Higham bound
 * helper). Real data only. */
int oracle_contract_abs(int na, const int64_t *sa, const int32_t *la, const double *A,
                        int nb, const int64_t *sb, const int32_t *lb, const double *B,
                        int nc, const int32_t *lc, double *C, int nthreads) {
  int64_t na_el = prod(na, sa), nb_el = prod(nb, sb);
  double *aa = (double *)malloc((size_t)na_el * sizeof(double));
  double *bb = (double *)malloc((size_t)nb_el * sizeof(double));
  if (!aa || !bb) { free(aa); free(bb); return OR_NOMEM; }
  for (int64_t i = 0; i < na_el; i++) aa[i] = A[i] < 0 ? -A[i] : A[i];
  for (int64_t i = 0; i < nb_el; i++) bb[i] = B[i] < 0 ? -B[i] : B[i];
  int st = oracle_contract(0, na, sa, la, aa, nb, sb, lb, bb, nc, lc, C, nthreads);
  free(aa); free(bb);
  return st;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
