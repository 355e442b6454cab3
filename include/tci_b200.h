/*
 * tci_b200.h -- C ABI of libtci_b200.so, the B200 (sm_100a) hot path beneath
 * the Tensor Computing Interface (TCI) of arXiv:2512.23917.
 *
 * Citations: "P:n" = PAPER.md line n of the paper's LaTeX source (section /
 * equation named beside it). Readings of ambiguous passages are numbered
 * R1..R24 in DESIGN.md section "Readings".
 *
 * General conventions (apply to every entry point):
 *  - Memory layout: row-major, last bond index fastest (R1). A
 *    tensor descriptor describes a dense row-major array; complex elements
 *    are interleaved (re, im), as in C99 _Complex / std::complex / torch.
 *  - Ownership: element memory is ALWAYS owned by the caller (e.g. torch
 *    tensors). The library never allocates device memory on a compute call;
 *    scratch comes from tci_workspace_attach. Descriptors (tci_tensor_t) and
 *    contexts (tci_ctx_t) are library-allocated and freed by
 *    tci_tensor_free / tci_destroy_context.
 *  - Asynchrony: compute calls enqueue kernels on the context's CUDA stream
 *    and return; results are visible to work ordered after them on that
 *    stream. Launch failures return TCI_ERR_CUDA; asynchronous device faults
 *    surface on a later call or on tci_synchronize.
 *  - Errors: every fallible call returns one tci_status_t; arguments are
 *    validated completely BEFORE any kernel is launched, so an error leaves
 *    all outputs untouched. tci_last_error() returns a thread-local message
 *    for the most recent failure.
 *  - Diagnostics: TCI_VERBOSE is read once at context creation:
 *    0 silent; 1 one line per call on stderr
 *    "tci:<op> shapes=[d0,d1;e0,...] dtype=<r32|r64|c64|c128>";
 *    2 additionally " time_us=<int>" (the call synchronizes its stream).
 *  - Thread safety: one context must not be used by two host threads at
 *    once; distinct contexts are independent.
 */
#ifndef TCI_B200_H
#define TCI_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TCI_API __attribute__((visibility("default")))
#else
#define TCI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Handle to the back-end context (Tab. III "context_handle_t", P:656;
 * create/destroy P:2332-2373). Owns the CUDA stream binding, the attached
 * workspace, the plan cache and (optionally) an NCCL communicator. */
typedef struct tci_ctx_s *tci_ctx_t;

/* Tensor descriptor (Tab. III "ten_t"; tensor definition section
 * II.A P:115-146): dtype + order + shape over BORROWED memory. */
typedef struct tci_tensor_s *tci_tensor_t;

/* Element type: the scalar field K in {R, C} at single or double
 * precision (Tab. III "elem_t"; reading R14). */
typedef enum {
  TCI_R32 = 1,   /* float                               4 B */
  TCI_R64 = 2,   /* double                              8 B */
  TCI_C64 = 3,   /* complex float,  interleaved (re,im) 8 B */
  TCI_C128 = 4   /* complex double, interleaved (re,im) 16 B */
} tci_dtype_t;

/* Status codes (the first kinds follow SPEC.md's
 * taxonomy, the rest are build-specific). */
typedef enum {
  TCI_OK = 0,
  TCI_ERR_SHAPE_MISMATCH = 1,   /* equal labels with different dims; wrong output shape; reshape size change */
  TCI_ERR_ORDER_MISMATCH = 2,   /* label string length != tensor order; permutation length != order */
  TCI_ERR_OUT_OF_RANGE = 3,     /* a dimension < 1 (R13); rank/index out of range */
  TCI_ERR_LABEL_CONFLICT = 4,   /* repeated label in one operand or in gamma; label in all
                                   three lists (R3); label in one input only and not in gamma (R4);
                                   gamma label absent from the inputs (R5) */
  TCI_ERR_PARSE = 5,            /* unparseable label string (NUL-terminated string expected) */
  TCI_ERR_DEAD_CONTEXT = 6,     /* call on a destroyed context */
  TCI_ERR_UNSUPPORTED = 7,      /* dtype mismatch between operands (one TenT per call);
                                   order > 16; host memory passed to a compute call */
  TCI_ERR_INVALID_ARGUMENT = 8, /* NULL pointer, not a permutation, bad enum value */
  TCI_ERR_WORKSPACE = 9,        /* attached workspace smaller than the call needs */
  TCI_ERR_CUDA = 10,            /* a CUDA runtime error (message in tci_last_error) */
  TCI_ERR_NCCL = 11             /* an NCCL error, or no communicator initialised */
} tci_status_t;

#define TCI_MAX_ORDER 16

/* ---------------------------------------------------------------------- */
/* Context and version                         */
/* ---------------------------------------------------------------------- */

/* "M.m" version string of the TCI specification implemented: "1.0"
 * (P:2505-2517). Static storage; never fails. */
TCI_API const char *tci_version(void);

/* Create a context bound to CUDA `device` and CUDA stream `stream`
 * (a cudaStream_t passed as void*; NULL = the legacy default stream).
 * The stream stays owned by the caller and must outlive the context.
 * Reads TCI_VERBOSE once.
 * Errors: INVALID_ARGUMENT (ctx NULL), OUT_OF_RANGE (no such device), CUDA. */
TCI_API tci_status_t tci_create_context(tci_ctx_t *ctx, int device, void *stream);

/* Destroy a context: releases descriptors' bookkeeping, the
 * plan cache and the NCCL communicator. Never frees caller memory (the
 * attached workspace included). The handle stays "dead" (not freed) so
 * that any later call -- a second destroy included -- returns
 * DEAD_CONTEXT. */
TCI_API tci_status_t tci_destroy_context(tci_ctx_t ctx);

/* Block the host until all work enqueued on the context stream finished.
 * Errors: DEAD_CONTEXT, CUDA (including sticky asynchronous faults). */
TCI_API tci_status_t tci_synchronize(tci_ctx_t ctx);

/* CUDA-graph capture of a call sequence (host-path latency of short chains,
 * e.g. config 1's 20 small contracts; PAPER.md:473 notes the per-call
 * overhead at small bond dimensions). Between tci_graph_begin and
 * tci_graph_end the calls on this context record their kernels into a CUDA
 * graph (stream capture of the context stream, thread-local mode) instead
 * of running them; tci_graph_launch replays the recorded kernels on the
 * context stream with the same pointers and shapes (the caller keeps the
 * tensors and the attached workspace alive and unchanged in size). Calls
 * that synchronize or read results on the host (Lanczos, SVD, guard
 * statistics, profiling, staged copies) fail inside a capture; so does a
 * workspace that would need to grow. tci_graph_end always ends the capture.
 * The context stream must be a created stream: the legacy NULL stream
 * cannot be captured (INVALID_ARGUMENT).
 * Errors: DEAD_CONTEXT, INVALID_ARGUMENT (NULL out / not capturing / already
 * capturing / legacy NULL stream), CUDA (an illegal call during capture
 * invalidates it). */
typedef struct tci_graph_s *tci_graph_t;
TCI_API tci_status_t tci_graph_begin(tci_ctx_t ctx);
TCI_API tci_status_t tci_graph_end(tci_ctx_t ctx, tci_graph_t *graph);
TCI_API tci_status_t tci_graph_launch(tci_ctx_t ctx, tci_graph_t graph);
TCI_API tci_status_t tci_graph_destroy(tci_graph_t graph);

/* Thread-local message describing the last failed call on this thread
 * ("" if none). Static thread-local storage; valid until the next call. */
TCI_API const char *tci_last_error(void);

/* complex128 GEMM algorithm of a context:
 *  TCI_GEMM_DMMA_3M (default): FP64 tensor cores (DMMA), Gauss 3-multiplication
 *    complex product;
 *  TCI_GEMM_DMMA_4M: DMMA, textbook 4-multiplication product;
 *  TCI_GEMM_OZAKI_INT8: Ozaki-II integer-modular emulation on the INT8 tcgen05
 *    tensor cores (exact power-of-two K-balancing A diag(2^s), diag(2^-s) B,
 *    row/column scaling to t >= 46-bit integers, exact residue GEMMs, exact
 *    CRT), used for GEMMs of >= 4e9 complex MACs; needs more scratch (the
 *    *_workspace_size queries account for it). Each such GEMM is guarded
 *    (tci_set_ozaki_guard): when its estimated relative Frobenius truncation
 *    error exceeds the context tolerance it is recomputed on DMMA.
 * The initial value comes from TCI_ZGEMM_ALGO = 3m | 4m | ozaki (read at
 * context creation). Setting it synchronizes the context stream. */
#define TCI_GEMM_DMMA_3M 0
#define TCI_GEMM_DMMA_4M 1
#define TCI_GEMM_OZAKI_INT8 2
TCI_API tci_status_t tci_set_gemm_algorithm(tci_ctx_t ctx, int algo);

/* Diagnostic (pure host): the Ozaki parameters for contraction length K --
 * number of moduli *nmod, integer bit budget *t (operands are scaled to
 * |A'| < 2^t), and the moduli (moduli[nmod], may be NULL). Returns 0, or
 * OUT_OF_RANGE when K is outside 1..131072 (the int32 exactness limit). */
TCI_API int tci_ozaki_params(int64_t K, int *nmod, int *t, int *moduli);

/* Complex128 Ozaki-II variant of a context (reading R33):
 *  TCI_OZAKI_CPLX_GAUSS (default): Gaussian moduli -- odd, pairwise coprime,
 *    every prime factor = 1 mod 4 -- each with a root j_l, j_l^2 = -1 (mod
 *    m_l); a + ib is mapped to (a + j_l b, a - j_l b) mod m_l, a ring
 *    homomorphism Z[i] -> Z_m x Z_m, so a complex product modulo m_l is two
 *    INT8 residue GEMMs (15 moduli -> 30 GEMMs for K <= ~69k);
 *  TCI_OZAKI_CPLX_3M: the float64 moduli with the 3M split (P = ArBr,
 *    Q = AiBi, S = (Ar+Ai)(Br+Bi)): three GEMMs per modulus (14 -> 42).
 * Both are exact up to the same operand truncation (R26). The initial value
 * comes from TCI_OZAKI_CPLX = gauss | 3m (read at context creation).
 * Synchronizes the context stream. Errors: DEAD_CONTEXT, INVALID_ARGUMENT. */
/* Float32 / complex64 GEMM algorithm of a context (reading R34):
 *  TCI_F32_OZAKI_INT8 (default): GEMMs of >= 4e9 MACs run the Ozaki-II scheme
 *    on the INT8 tcgen05 tensor cores with a bit budget t >= 24 (8-9 moduli
 *    real, 9-10 Gaussian complex): operand entries within a factor 2 of their
 *    line maximum are exact, the integer products and sums are exact, the
 *    result is rounded once to float32. Guarded like the float64 path, with
 *    tolerance max(guard tol, 1e-7); a flagged GEMM is recomputed on the FP64
 *    cores;
 *  TCI_F32_FP64_CORES: products and sums in float64 on the CUDA cores (R20).
 * The initial value comes from TCI_F32_ALGO = ozaki | fp64 (context
 * creation). Synchronizes the context stream. Errors: DEAD_CONTEXT,
 * INVALID_ARGUMENT. */
/* Diagnostic (pure host): the Ozaki parameters of float32 (cplx = 0) or
 * complex64 (cplx != 0, Gaussian moduli) GEMMs for contraction length K:
 * moduli count, bit budget t (>= 24), moduli[<= 16], residue planes per
 * modulus (1 or 2). Out-pointers may be NULL. Returns 0 or OUT_OF_RANGE. */
TCI_API int tci_ozaki_params_f32(int64_t K, int cplx, int *nmod, int *t, int *moduli, int *planes_per_mod);
#define TCI_F32_OZAKI_INT8 0
#define TCI_F32_FP64_CORES 1
TCI_API tci_status_t tci_set_f32_algorithm(tci_ctx_t ctx, int algo);

#define TCI_OZAKI_CPLX_GAUSS 0
#define TCI_OZAKI_CPLX_3M 1
TCI_API tci_status_t tci_set_ozaki_complex(tci_ctx_t ctx, int variant);

/* Diagnostic (pure host): the parameters of the complex128 Ozaki GEMMs of
 * `variant` for contraction length K: moduli count, bit budget t, moduli,
 * the roots j_l (Gaussian; 0 for 3M) and the residue planes per modulus
 * (2 Gaussian, 3 3M). Arrays hold up to 16 entries; any out-pointer may be
 * NULL. Returns 0, INVALID_ARGUMENT for an unknown variant, or OUT_OF_RANGE
 * when K is outside 1..131072. */
TCI_API int tci_ozaki_params_complex(int64_t K, int variant, int *nmod, int *t, int *moduli, int *roots,
                                     int *planes_per_mod);
TCI_API tci_status_t tci_get_gemm_algorithm(tci_ctx_t ctx, int *algo);

/* Accuracy guard of the Ozaki-II GEMMs (reading R26; the north
 * star's 1e-12 relative-Frobenius bar). Entry (m,k) of A is rounded to an
 * integer at scale 2^(t - E_m + s_k), so its error is eps 2^(E_m - t - s_k),
 * |eps| <= 1/2 per real component. With independent errors
 *   est^2 = c 4^-t (sum_m 4^E_m ||B'||_F^2 + ||A'||_F^2 sum_n 4^E_n) / ||C||_F^2
 * (c = 1/6 complex, 1/12 real; A' = A diag(2^s), B' = diag(2^-s) B) is the
 * expected squared relative Frobenius error; it is evaluated on the device
 * after the CRT and, when est > tol, the GEMM is recomputed on DMMA (a
 * launch gated by a device flag: no host synchronisation). tol <= 0 turns
 * the guard off. Default 1e-13 (TCI_OZAKI_GUARD=0 at context creation: off).
 * Errors: DEAD_CONTEXT, INVALID_ARGUMENT (NaN). */
TCI_API tci_status_t tci_set_ozaki_guard(tci_ctx_t ctx, double tol);

/* Statistics of the guard since context creation or the last reset
 * (synchronizes the context stream): Ozaki GEMMs checked, how many were
 * recomputed on DMMA, how many ran with a non-trivial K-balancing, the last
 * and the maximum estimate. Any out-pointer may be NULL; reset != 0 zeroes
 * the counters after reading. Errors: DEAD_CONTEXT, CUDA. */
TCI_API tci_status_t tci_ozaki_guard_stats(tci_ctx_t ctx, int reset, int64_t *gemms, int64_t *fallbacks,
                                           int64_t *balanced, double *last_est, double *max_est);

/* Attach caller-owned device scratch memory of `bytes` bytes (256-byte
 * aligned pointer). Replaces any previous attachment; NULL/0 detaches. Calls
 * that need scratch (tci_contract with permutes or aliasing, tci_heff_apply)
 * return WORKSPACE if it is too small, before launching anything. */
TCI_API tci_status_t tci_workspace_attach(tci_ctx_t ctx, void *dev_ws, size_t bytes);

/* ---------------------------------------------------------------------- */
/* Tensor descriptors and queries                              */
/* ---------------------------------------------------------------------- */

/* Describe `data` as a row-major tensor of `order` bonds with dimensions
 * shape[0..order-1] (each >= 1, R13; order 0 = scalar with one element).
 * `data` is borrowed: device memory (cudaMalloc / torch CUDA tensor) for
 * compute calls; host memory is accepted for descriptors used only with
 * tci_copy (pinned host memory for asynchronous copies). The location is
 * detected with cudaPointerGetAttributes. Needs 16-byte-aligned `data` for
 * complex128; element alignment otherwise.
 * Errors: INVALID_ARGUMENT, UNSUPPORTED (order > 16), OUT_OF_RANGE (dim < 1),
 * DEAD_CONTEXT. */
TCI_API tci_status_t tci_tensor_create(tci_ctx_t ctx, tci_dtype_t dtype, int order,
                               const int64_t *shape, void *data, tci_tensor_t *out);

/* Free a descriptor (never the element memory). */
TCI_API tci_status_t tci_tensor_free(tci_ctx_t ctx, tci_tensor_t t);

TCI_API tci_status_t tci_order(tci_ctx_t ctx, tci_tensor_t t, int *order);
TCI_API tci_status_t tci_shape(tci_ctx_t ctx, tci_tensor_t t, int64_t *shape);         /* P:766-783, shape[order] */
TCI_API tci_status_t tci_size(tci_ctx_t ctx, tci_tensor_t t, int64_t *n);              /* P:786-803, elements */
TCI_API tci_status_t tci_size_bytes(tci_ctx_t ctx, tci_tensor_t t, int64_t *bytes);

/* Copy all elements of `src` into `dst` (same dtype and same element count;
 * shapes may differ as by reshape) on the context stream; either side may be
 * host or device memory (cudaMemcpyAsync). Used for end-to-end host I/O. */
TCI_API tci_status_t tci_copy(tci_ctx_t ctx, tci_tensor_t src, tci_tensor_t dst);

/* Asynchronous lanes (the asynchronous API the paper defers to a later
 * revision): lane 0 is the context stream (every compute call),
 * lanes 1 and 2 are library-owned copy streams (host -> device and device ->
 * host traffic, so both PCIe directions and the compute can run at once).
 * tci_copy_async enqueues tci_copy's copy on `lane`; tci_lane_record records
 * event `slot` (0..15) on `lane`; tci_lane_wait makes `lane` wait for the
 * last record of `slot` (on any lane). With these a caller double-buffers
 * device inputs: the copies of step i+1 run while step i computes.
 * Errors: OUT_OF_RANGE (lane, slot), as tci_copy, CUDA. */
TCI_API tci_status_t tci_copy_async(tci_ctx_t ctx, tci_tensor_t src, tci_tensor_t dst, int lane);
TCI_API tci_status_t tci_lane_record(tci_ctx_t ctx, int lane, int slot);
TCI_API tci_status_t tci_lane_wait(tci_ctx_t ctx, int lane, int slot);

/* ---------------------------------------------------------------------- */
/* Manipulation: reshape and transpose (Eq. (1)) */
/* ---------------------------------------------------------------------- */

/* In-place reshape: metadata only, element order in memory preserved
 * (P:1170-1171). Errors: SHAPE_MISMATCH (element count changes),
 * OUT_OF_RANGE (dim < 1), UNSUPPORTED (order > 16). Launches nothing. */
TCI_API tci_status_t tci_reshape(tci_ctx_t ctx, tci_tensor_t inout, int order,
                         const int64_t *new_shape);

/* Out-of-place transpose, Eq. (1): out bond k is in bond
 * new_order[k], out.shape[k] = in.shape[new_order[k]] (reading R2, NumPy
 * axes semantics). `out` must have exactly that shape and in's dtype; in and
 * out must not overlap. Bitwise exact (pure data movement). Kernel: shared-
 * memory tiled transpose with 16-byte coalesced loads/stores (HBM-bound).
 * Errors: ORDER_MISMATCH, INVALID_ARGUMENT (not a permutation / overlap),
 * SHAPE_MISMATCH, UNSUPPORTED, CUDA. */
TCI_API tci_status_t tci_permute(tci_ctx_t ctx, tci_tensor_t in, const int32_t *new_order,
                         tci_tensor_t out);

/* ---------------------------------------------------------------------- */
/* contract (Eq. (3))                               */
/* ---------------------------------------------------------------------- */

/* Shape of c for labels la (order(a) entries), lb (order(b)), lc (nc):
 * shape_c[k] = dim of label lc[k]. Validates exactly like tci_contract.
 * Launches nothing. */
TCI_API tci_status_t tci_contract_out_shape(tci_ctx_t ctx, tci_tensor_t a, const int32_t *la,
                                    tci_tensor_t b, const int32_t *lb, int nc,
                                    const int32_t *lc, int64_t *shape_c);

/* Label-based Einstein contraction, list API:
 *   c[gamma] = sum over S of a[alpha] * b[beta],  S = alpha ∩ beta \ gamma,
 * gamma = lc gives the free bonds of c and their order;
 * equal labels must have equal dims; empty gamma (order(c)=0)
 * gives a 1-element result; c may alias a and/or b -- the
 * library then computes into workspace and copies. No implicit conjugation
 * (R9). a, b, c: same dtype, device memory; c pre-created with the exact
 * output shape (see tci_contract_out_shape). Lowered to permute -> GEMM
 * over the fused contracted legs -> permute back, with the
 * permutes folded into the GEMM loaders/epilogue whenever the legs fuse.
 * Label arrays are read during the call only.
 * Errors: LABEL_CONFLICT, SHAPE_MISMATCH, UNSUPPORTED, WORKSPACE, CUDA,
 * DEAD_CONTEXT, INVALID_ARGUMENT. */
TCI_API tci_status_t tci_contract(tci_ctx_t ctx, tci_tensor_t a, const int32_t *la,
                          tci_tensor_t b, const int32_t *lb,
                          tci_tensor_t c, const int32_t *lc);

/* String API: NUL-terminated strings, one byte per label
 * (unsigned char value, case-sensitive; reading R12); each string must have
 * exactly order(tensor) bytes, else ORDER_MISMATCH. "" is the empty list. */
TCI_API tci_status_t tci_contract_str(tci_ctx_t ctx, tci_tensor_t a, const char *la,
                              tci_tensor_t b, const char *lb,
                              tci_tensor_t c, const char *lc);

/* Workspace bytes tci_contract needs for these operands (0 when no
 * permute/aliasing copy is needed). */
TCI_API tci_status_t tci_contract_workspace_size(tci_ctx_t ctx, tci_tensor_t a, const int32_t *la,
                                         tci_tensor_t b, const int32_t *lb,
                                         tci_tensor_t c, const int32_t *lc, size_t *bytes);

/* ---------------------------------------------------------------------- */
/* Chains (definitions DESIGN.md R15-R18; the paper has no text for them)  */
/* ---------------------------------------------------------------------- */

/* Two-site DMRG effective Hamiltonian apply (R15; DMRG cited
 * P:55):
 *   out[b,p,q,e] = sum L[a,w,b] psi[a,s,t,c] W1[w,v,s,p] W2[v,x,t,q] R[c,x,e]
 * Shapes: L (chi_l, D, chi_lo), W1 (D, D1, d, d), W2 (D1, D2, d, d),
 * R (chi_r, D2, chi_ro), psi (chi_l, d, d, chi_r), out (chi_lo, d, d, chi_ro).
 * W index order: (left MPO bond, right MPO bond, ket/in phys, bra/out phys).
 * dtype r64 or c128 (all operands equal). The FLOP-optimal pairwise order is
 * chosen by the chain planner (a7): L.psi (GEMM) -> W1,W2 (skinny kernel,
 * fused as W12 when cheaper) -> .R (GEMM); intermediates live in the
 * attached workspace (tci_heff_workspace_size). Sharding (8(e)): pass the
 * rank's slice L[:, :, b_r] (chi_lo = chi/P) and its out slab; the result is
 * bitwise identical to the unsharded rows.
 * Errors: SHAPE_MISMATCH, UNSUPPORTED, WORKSPACE, CUDA, DEAD_CONTEXT. */
TCI_API tci_status_t tci_heff_workspace_size(tci_ctx_t ctx, tci_dtype_t dtype, int64_t chi_l,
                                     int64_t chi_lo, int64_t chi_r, int64_t chi_ro,
                                     int64_t d, int64_t D, int64_t D1, int64_t D2,
                                     size_t *bytes);
TCI_API tci_status_t tci_heff_apply(tci_ctx_t ctx, tci_tensor_t L, tci_tensor_t W1,
                            tci_tensor_t W2, tci_tensor_t R, tci_tensor_t psi,
                            tci_tensor_t out);

/* TEBD two-site gate application (R16; iTEBD of P:392-403):
 *   theta[lt] = sum_{s,t} U[p,q,s,t] sum_b A[la] B[lb]
 * with la a permutation of "asb", lb of "btc", lu == "pqst" (gate rows =
 * out (p,q), cols = in (s,t), R16) and lt a permutation of "apqc" (same
 * label letters as documented; any byte values are accepted as long as the
 * roles match by position in the canonical strings "asb","btc","pqst","apqc"
 * -- i.e. the call maps la/lb/lt onto those roles by label identity).
 * When the physical legs are adjacent to the bond legs as in the natural
 * ("asb","btc","apqc") or physical-first ("sab","tbc","paqc") layouts, the
 * gate is applied in the GEMM epilogue (no intermediate theta pass).
 * Errors: LABEL_CONFLICT, SHAPE_MISMATCH, UNSUPPORTED, WORKSPACE, CUDA. */
TCI_API tci_status_t tci_tebd_theta(tci_ctx_t ctx, tci_tensor_t A, const char *la,
                            tci_tensor_t B, const char *lb,
                            tci_tensor_t U, const char *lu,
                            tci_tensor_t theta, const char *lt);

/* Scratch bytes tci_tebd_theta needs for these operands under the context's
 * GEMM algorithm (0 for the fused DMMA gate epilogue; the intermediate A.B +
 * the contraction's scratch otherwise, incl. the Ozaki residue planes).
 * Reads only descriptors. Errors: as tci_tebd_theta's validation. */
TCI_API tci_status_t tci_tebd_workspace_size(tci_ctx_t ctx, tci_tensor_t A, const char *la, tci_tensor_t B,
                                             const char *lb, tci_tensor_t U, const char *lu, tci_tensor_t theta,
                                             const char *lt, size_t *bytes);

/* Environment update (R28): the DMRG step before
 * every H_eff, with the index conventions of tci_heff_apply (E[ket bond, MPO
 * bond, bra bond]; W[w_left, w_right, s = ket physical, t = bra physical]):
 *   side 0 (left):  out[b,v,e] = sum E[a,w,c] ket[a,s,b] W[w,v,s,t] conj(bra[c,t,e])
 *     E [chi_k, D, chi_b], ket [chi_k, d, chi_ko], W [D, Dv, d, d],
 *     bra [chi_b, d, chi_bo], out [chi_ko, Dv, chi_bo]
 *   side 1 (right): out[a,w,f] = sum ket[a,s,c] W[w,x,s,t] E[c,x,e] conj(bra[f,t,e])
 *     E [chi_k, D, chi_b], ket [chi_ko, d, chi_k], W [Dv, D, d, d],
 *     bra [chi_bo, d, chi_b], out [chi_ko, Dv, chi_bo]
 * (conj is the identity for r64). bra may be the same tensor as ket
 * (<psi|H|psi>). Executed as GEMM (E.ket, contract engine) -> skinny MPO pass
 * -> conj(bra) (one HBM pass into workspace) -> GEMM, permute-free;
 * intermediates live in the attached workspace (tci_env_workspace_size).
 * All device tensors, one dtype (r64 or c128); out must not overlap inputs.
 * Errors: INVALID_ARGUMENT (side, overlap), ORDER_MISMATCH, SHAPE_MISMATCH,
 * UNSUPPORTED (dtype; D*d or Dv*d > 128), WORKSPACE, CUDA, DEAD_CONTEXT. */
TCI_API tci_status_t tci_env_workspace_size(tci_ctx_t ctx, int side, tci_tensor_t E, tci_tensor_t ket,
                                            tci_tensor_t W, tci_tensor_t bra, tci_tensor_t out, size_t *bytes);
TCI_API tci_status_t tci_env_update(tci_ctx_t ctx, int side, tci_tensor_t E, tci_tensor_t ket, tci_tensor_t W,
                                    tci_tensor_t bra, tci_tensor_t out);

/* Elementwise complex conjugation (tci::cplx_conj): out[i] =
 * conj(in[i]). out == in conjugates in place (overload (1)); otherwise out
 * must not overlap in (overload (2)). Real data: in place is a no-op, out of
 * place a deep copy. Same dtype / shape required. Asynchronous on
 * the context stream; bitwise exact.
 * Errors: UNSUPPORTED (dtype mismatch, complex64), ORDER_MISMATCH,
 * SHAPE_MISMATCH, INVALID_ARGUMENT (partial overlap), CUDA, DEAD_CONTEXT. */
TCI_API tci_status_t tci_cplx_conj(tci_ctx_t ctx, tci_tensor_t in, tci_tensor_t out);

/* ---------------------------------------------------------------------- */
/* Vector functions (device kernels, deterministic reductions) and the     */
/* Lanczos driver around H_eff                              */
/* ---------------------------------------------------------------------- */

/* Frobenius norm (Eq. frob_norm) into *out (host). r64/c128.
 * Synchronizes the context stream. Bitwise reproducible. */
TCI_API tci_status_t tci_norm(tci_ctx_t ctx, tci_tensor_t t, double *out);

/* In-place normalize to unit Frobenius norm; the original norm goes to
 * *norm_out (may be NULL). Zero norm -> INVALID_ARGUMENT. */
TCI_API tci_status_t tci_normalize(tci_ctx_t ctx, tci_tensor_t inout, double *norm_out);

/* out = s * in with s = s_re + i s_im (s_im must be 0 for real data)
 * (P:1784-1808). out may be in (in-place overload (1)). */
TCI_API tci_status_t tci_scale(tci_ctx_t ctx, tci_tensor_t in, double s_re, double s_im, tci_tensor_t out);

/* out = sum_{i<m} s_i ins[i]; coefs = m (re, im) pairs, or
 * NULL for all s_i = 1 (overload (1)); all shapes identical; out may alias
 * any input. */
TCI_API tci_status_t tci_linear_combine(tci_ctx_t ctx, int m, const tci_tensor_t *ins, const double *coefs,
                                        tci_tensor_t out);

/* <a|b> = sum_i conj?(a_i) b_i into out[2] = (re, im): the full contraction
 * to a scalar of section III, with cplx_conj of a
 * when conj_a != 0. Synchronizes. */
TCI_API tci_status_t tci_inner(tci_ctx_t ctx, tci_tensor_t a, tci_tensor_t b, int conj_a, double *out);

/* Lowest eigenpair of H_eff (tci_heff_apply operator; Hermitian by the
 * caller's construction) by Lanczos with full re-orthogonalisation: psi is
 * the start vector on entry and the normalised Ritz vector on return;
 * *energy = lowest Ritz value; *iters = Krylov dimension used. Stops when
 * the Ritz value moves by < tol or the residual vanishes, at most max_iter
 * (1..512) steps. With a communicator (tci_comm_init, nranks P) L is this
 * rank's slice L[:, :, b_r] (chi_l / P columns) and each step ends with one
 * NCCL all-gather of the output slabs; every rank then holds identical
 * vectors. Workspace: tci_lanczos_workspace_size (heff scratch + (max_iter+2)
 * vectors). Host synchronizes once per inner product. */
TCI_API tci_status_t tci_lanczos_workspace_size(tci_ctx_t ctx, tci_tensor_t L, tci_tensor_t W1, tci_tensor_t W2,
                                                tci_tensor_t R, tci_tensor_t psi, int max_iter, size_t *bytes);
TCI_API tci_status_t tci_heff_lanczos(tci_ctx_t ctx, tci_tensor_t L, tci_tensor_t W1, tci_tensor_t W2,
                                      tci_tensor_t R, tci_tensor_t psi, int max_iter, double tol, double *energy,
                                      int *iters);

/* MPS overlap / norm transfer chain (R17; the section III overlap
 * by contraction): with E_0 = [[1]],
 *   E_{i+1}[y,w] = sum_{x,z,s} E_i[x,z] bra_i[x,s,y] ket_i[z,s,w],
 * out = E_n of shape (bra[n-1].shape[2], ket[n-1].shape[2]). Bilinear (no
 * conjugation, R9). bra[i], ket[i]: order-3 site tensors [left, phys, right]
 * (device, r64 or c128), bra[0]/ket[0] left bond 1, physical dims equal per
 * site. Executed as ONE single-CTA kernel with E and X in shared memory (the
 * chain is launch-latency bound, config 1); bonds <= 32, d <= 4, n <= 64,
 * else UNSUPPORTED (use tci_contract for larger chains).
 * Errors: ORDER_MISMATCH, SHAPE_MISMATCH, UNSUPPORTED, OUT_OF_RANGE, CUDA. */
TCI_API tci_status_t tci_mps_overlap(tci_ctx_t ctx, int n, const tci_tensor_t *bra,
                                     const tci_tensor_t *ket, tci_tensor_t out);

/* ---------------------------------------------------------------------- */
/* Multi-GPU (8(e)): one communicator per context                          */
/* ---------------------------------------------------------------------- */

/* Initialise the context's NCCL communicator from a 128-byte ncclUniqueId
 * (broadcast by the caller, e.g. with torch.distributed) for `nranks` ranks.
 * Errors: OUT_OF_RANGE (rank), NCCL, DEAD_CONTEXT. */
TCI_API tci_status_t tci_comm_init(tci_ctx_t ctx, const void *nccl_unique_id, int nranks, int rank);

/* Fill `id` (128 bytes) with a new ncclUniqueId (rank 0 calls this). */
TCI_API tci_status_t tci_comm_unique_id(void *id);

/* All-gather along the slowest bond: full = concat over ranks (rank order)
 * of each rank's `shard` (ncclAllGather on the context stream). full must
 * have nranks * size(shard) elements of the same dtype.
 * Errors: NCCL (no communicator), SHAPE_MISMATCH, UNSUPPORTED. */
TCI_API tci_status_t tci_allgather(tci_ctx_t ctx, tci_tensor_t shard, tci_tensor_t full);

/* Peer-memory all-gather fused into the H_eff output (the one exchange of
 * the sharded apply). One process per GPU. Each
 * rank owns (caller-allocated device memory) its full output buffer
 * [P * chi_lo_r, d, d, chi_ro] (complex128 / float64, 16-byte aligned) and a
 * zeroed flag array of P uint32; it exports both with tci_ipc_handle, the
 * ranks exchange the (handle, offset) pairs (e.g. with
 * torch.distributed.all_gather_object), map the peers' with tci_ipc_open and
 * register the P pointers of each kind (own ones included, rank order) with
 * tci_gather_register.
 *
 * tci_ipc_handle: `handle` receives the 64-byte cudaIpcMemHandle_t of the
 * allocation holding dev_ptr, `offset` dev_ptr's offset in it.
 * tci_ipc_open: maps a peer's allocation (cudaIpcOpenMemHandle, lazy peer
 * access) and returns base + offset; tci_ipc_close unmaps it.
 * Errors: INVALID_ARGUMENT (NULL, not a device allocation, unknown pointer),
 * CUDA. */
TCI_API tci_status_t tci_ipc_handle(const void *dev_ptr, void *handle, size_t *offset);
TCI_API tci_status_t tci_ipc_open(const void *handle, size_t offset, void **dev_ptr);
TCI_API tci_status_t tci_ipc_close(void *dev_ptr);

/* Register the gather's pointer tables (nranks <= 8): full[i] / flags[i] are
 * rank i's buffers, valid in this process. Errors: OUT_OF_RANGE, INVALID_ARGUMENT. */
TCI_API tci_status_t tci_gather_register(tci_ctx_t ctx, int nranks, int rank, void *const *full,
                                         void *const *flags);

/* H_eff psi on this rank's slab (L = L[:, :, b_r], chi_lo_r columns) with the
 * result gathered into EVERY rank's `full` (the registered buffer): rows
 * [r chi_lo_r, (r+1) chi_lo_r) of the slowest leg are this rank's. The Ozaki
 * GEMM4 epilogue stores each output element locally and into every peer's
 * buffer over NVLink (no separate collective); the DMMA path pushes the slab
 * after GEMM4 with a peer-copy kernel. A flag barrier (system-scope release /
 * acquire) before the chain and after the stores orders the steps across
 * ranks; on return (stream order) `full` holds the whole output on every
 * rank, bitwise equal to the unsharded tci_heff_apply. A barrier that waits
 * > 30 s sets an error flag read by tci_gather_status (synchronizes) instead
 * of hanging. With nranks = 1 it is tci_heff_apply into full.
 * Errors: as tci_heff_apply; INVALID_ARGUMENT if full is not the registered
 * buffer; SHAPE_MISMATCH if full's first leg != nranks x L's last leg. */
TCI_API tci_status_t tci_heff_apply_gather(tci_ctx_t ctx, tci_tensor_t L, tci_tensor_t W1, tci_tensor_t W2,
                                           tci_tensor_t R, tci_tensor_t psi, tci_tensor_t full);
TCI_API tci_status_t tci_gather_status(tci_ctx_t ctx, int *timed_out);

/* ---------------------------------------------------------------------- */
/* Diagnostics                                                             */
/* ---------------------------------------------------------------------- */

/* Number of CUDA kernels this context has launched so far (bench evidence). */
TCI_API tci_status_t tci_launch_count(tci_ctx_t ctx, int64_t *count);

/* Kernel profiling: when enabled, every GEMM / skinny / permute kernel the
 * context launches is bracketed by CUDA events recorded on the context
 * stream, together with its ALGORITHMIC work (GEMM: 2 flops per real MAC, 8
 * per complex MAC; bytes = operands read once + result written once).
 * Enabling (or disabling) synchronizes the stream and clears the records. */
TCI_API tci_status_t tci_profile_enable(tci_ctx_t ctx, int on);

/* Sum over recorded launches of `kind` (0 GEMM, 1 skinny, 2 permute,
 * 3 the INT8 tensor-core GEMMs inside Ozaki GEMMs -- "flops" = executed int8
 * ops, 2 per MAC):
 * launch count, total event time in ms, algorithmic flops and bytes.
 * Synchronizes the context stream. */
TCI_API tci_status_t tci_profile_query(tci_ctx_t ctx, int kind, int64_t *launches, double *ms,
                                       double *flops, double *bytes);

/* The H_eff order planner's decision (8(a7)) for the given dimensions:
 * writes the FLOP-optimal pairwise tree, e.g. "((((L.psi).W1).W2).R)", into
 * buf[n] and its multiply-add count into *macs. Returns 1 when the tree is
 * executed by the permute-free fast path, 0 when the generic tree executor
 * (contract calls) is used. Pure host computation. */
TCI_API int tci_heff_plan_tree(int64_t chi_l, int64_t chi_lo, int64_t chi_r, int64_t chi_ro,
                               int64_t d, int64_t D, int64_t D1, int64_t D2, char *buf, int n,
                               double *macs);

/* ---------------------------------------------------------------------- */
/* Singular value decomposition: tci::svd / tci::trunc_svd  */
/* ---------------------------------------------------------------------- */

/* Scratch bytes tci_svd / tci_trunc_svd need for a tensor of this dtype and
 * shape matricized with the first num_of_bds_as_row bonds as rows: two
 * working matrices of min(I,J) x max(I,J) and min(I,J)^2 elements (rounded
 * up to multiples of 32) plus O(min(I,J)) vectors.
 * Errors: UNSUPPORTED (dtype other than r64 / c128), OUT_OF_RANGE (k). */
TCI_API tci_status_t tci_svd_workspace_size(tci_ctx_t ctx, tci_dtype_t dtype, int order, const int64_t *shape,
                                            int num_of_bds_as_row, size_t *bytes);

/* tci::svd. a (order r, shape {d_0..d_{r-1}}, r64 or c128) is
 * matricized by grouping the first k = num_of_bds_as_row bonds into the row
 * index (1 <= k < r): A' is I x J, I = prod_{b<k} d_b, J = prod_{b>=k} d_b
 * (row-major, metadata only). A' = U S V^dagger with s_0 >= s_1 >= ... >=
 * s_{kappa-1} >= 0, kappa = min(I, J), folded back:
 *   u      [d_0, .., d_{k-1}, kappa]   dtype of a
 *   s_diag [kappa]                     r64 (real_ten_t), non-increasing
 *   v_dag  [kappa, d_k, .., d_{r-1}]   dtype of a
 * All three are caller-allocated device tensors of exactly these shapes;
 * none may overlap a; a is not modified. Scratch: tci_svd_workspace_size.
 * Method: block one-sided Jacobi on the FP64 tensor cores:
 * singular values to ~1e-14 relative to s_0, u and v_dag orthonormal to
 * ~1e-13; where s_i = 0 exactly the singular vector is completed to an
 * orthonormal set (R29). Synchronous (returns after the result is written).
 * Errors: UNSUPPORTED (dtype; u/v_dag dtype != a's, s_diag not r64),
 * OUT_OF_RANGE (k), ORDER_MISMATCH / SHAPE_MISMATCH (output descriptors),
 * INVALID_ARGUMENT (overlap), WORKSPACE, CUDA, DEAD_CONTEXT. */
TCI_API tci_status_t tci_svd(tci_ctx_t ctx, tci_tensor_t a, int num_of_bds_as_row, tci_tensor_t u,
                             tci_tensor_t s_diag, tci_tensor_t v_dag);

/* tci::trunc_svd, overload (2); overload (1) is chi_min = 1,
 * target_trunc_err = 0. The SVD as tci_svd, then the strategy of
 * P:2093-2098 on the pre-truncation s_0 >= .. >= s_{kappa-1}:
 *   a) discard all s_i < s_min; b) keep at least chi_min values, and if fewer
 *   remain after a) keep those; c) grow chi in descending order until
 *   eps <= target_trunc_err or chi = chi_max; chi >= 1 always (R30).
 * eps = sum_{i>=chi} s_i^2 / sum_i s_i^2 -> *trunc_err.
 * The output descriptors are passed with the CAPACITY shape, cap =
 * min(max(chi_min, chi_max), kappa) in the chi position (u [.., cap], s_diag
 * [cap], v_dag [cap, ..]); on success they are reshaped (metadata) to chi and
 * their buffers hold the dense row-major truncated tensors. *chi_out (may be
 * NULL) receives chi. Errors as tci_svd, plus OUT_OF_RANGE (chi_max < 1,
 * chi_min < 0, negative target_trunc_err or s_min). */
TCI_API tci_status_t tci_trunc_svd(tci_ctx_t ctx, tci_tensor_t a, int num_of_bds_as_row, tci_tensor_t u,
                                   tci_tensor_t s_diag, tci_tensor_t v_dag, double *trunc_err, int64_t chi_min,
                                   int64_t chi_max, double target_trunc_err, double s_min, int64_t *chi_out);

/* tci_heff_apply with the inputs in (pinned) host memory and the result
 * returned to host memory, copies overlapped with the computation: the
 * context's copy stream moves psi, W1, W2 to the device staging tensors
 * (L..out, device, caller-owned); GEMM1 starts when they have arrived and
 * reads L in eight column blocks, each copied in just before the Ozaki row
 * chunk (or DMMA row-block GEMM) that needs it; R is copied behind L while
 * GEMM1 and the MPO pass run; GEMM4's output rows are copied back in eight
 * chunks as they are finished. Equivalent to tci_copy x5,
 * tci_heff_apply, tci_copy, and stream-ordered on the context stream like
 * them (the context stream waits for the last D2H copy). Each *_h tensor
 * must match its device twin in dtype and shape (host or device memory;
 * pinned host memory for overlap). out_h may be NULL: the inputs are staged
 * in the same way and the result stays in `out`; the copies then do NOT wait
 * for work already queued on the context stream -- the caller orders copy
 * lane 1 (tci_lane_record / tci_lane_wait) so that `L`..`psi` are free, which
 * lets a stream of applies stage step i+1's inputs while step i computes. Errors: as
 * tci_heff_apply, plus SHAPE_MISMATCH for a twin mismatch. Scratch:
 * tci_heff_workspace_size. */
TCI_API tci_status_t tci_heff_apply_staged(tci_ctx_t ctx, tci_tensor_t L_h, tci_tensor_t W1_h, tci_tensor_t W2_h,
                                           tci_tensor_t R_h, tci_tensor_t psi_h, tci_tensor_t out_h,
                                           tci_tensor_t L, tci_tensor_t W1, tci_tensor_t W2, tci_tensor_t R,
                                           tci_tensor_t psi, tci_tensor_t out);

/* Compressed MPS-MPO application by zip-up (R32):
 * B ~ W|psi> for an open-boundary MPS A[i] [chi_{i-1}, d_i, chi_i] (chi_{-1} =
 * chi_{n-1} = 1) and MPO W[i] [D_{i-1}, D_i, d_i (in), d'_i (out)] (D_{-1} =
 * D_{n-1} = 1; index order of R15). Left to right: T1 = C.A_i, T = T1.W_i
 * (tci_contract semantics), then for i < n-1 the truncated SVD of T at
 * (k t)|(b v) (tci_trunc_svd with chi_min = 1, chi_max, target 0, s_min):
 * B_i = U, carry C = S V^dag; B_{n-1} = T. Every step runs in the library's
 * kernels; the host loops over the sites.
 * B[i] are caller-allocated device tensors of CAPACITY shape [c_{i-1}, d'_i,
 * c_i], c_{-1} = c_{n-1} = 1, c_i = min(chi_max, c_{i-1} d'_i, chi_i D_i); on
 * success their descriptors are reshaped to the kept bonds (dense row-major
 * buffers). *trunc_err = sum over bonds of the discarded weights.
 * With chi_max >= every exact bond and s_min = 0 the result is W|psi> exactly
 * (up to rounding). Synchronous. Scratch: tci_mps_mpo_zipup_workspace_size.
 * Errors: OUT_OF_RANGE (n < 1, chi_max < 1, s_min < 0), UNSUPPORTED (dtype),
 * ORDER_MISMATCH / SHAPE_MISMATCH (bonds, capacities), WORKSPACE, CUDA. */
TCI_API tci_status_t tci_mps_mpo_zipup_workspace_size(tci_ctx_t ctx, int n, const tci_tensor_t *A,
                                                      const tci_tensor_t *W, int64_t chi_max, size_t *bytes);
TCI_API tci_status_t tci_mps_mpo_zipup(tci_ctx_t ctx, int n, const tci_tensor_t *A, const tci_tensor_t *W,
                                       tci_tensor_t *B, int64_t chi_max, double s_min, double *trunc_err);

/* Diagnostics of the last tci_svd / tci_trunc_svd on this context: Jacobi
 * sweeps executed and the final sweep's largest relative off-diagonal
 * |<x_i|x_j>| / (|x_i| |x_j|) (convergence: <= max(1e-13, 4 sqrt(max(I,J)) eps),
 * env TCI_SVD_TOL overrides). */
TCI_API tci_status_t tci_svd_info(tci_ctx_t ctx, int *sweeps, double *off);

#ifdef __cplusplus
}
#endif
#endif /* TCI_B200_H */
