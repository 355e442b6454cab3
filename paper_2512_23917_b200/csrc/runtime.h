// runtime.h -- host-side runtime structures of libtci_b200 (context, tensor
// descriptors, error reporting, planner entry points). Internal.
#pragma once
#include <cstdarg>
#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "tci_internal.h"

struct tci_ctx_s {
  uint32_t magic;
  bool alive;
  int device;
  cudaStream_t stream;
  int verbose;
  void *ws;
  size_t ws_bytes;
  int64_t launches;
  void *nccl_comm;
  int nranks, rank;
  // kernel profiling (tci_profile_enable): CUDA events on the context stream
  // around every GEMM / skinny / permute launch, with algorithmic work
  bool prof_on;
  struct ProfRec {
    int kind;
    cudaEvent_t a, b;
    double flops, bytes;
  };
  std::vector<ProfRec> prof;
  // plan cache: key -> serialized plan decision (see contract.cpp)
  std::unordered_map<std::string, std::vector<int64_t>> plan_cache;
  int64_t plan_hits, plan_misses;
  int zgemm_algo;       // complex128 GEMM algorithm (kZ3M default; tci_set_gemm_algorithm)
  int f32_algo;         // float32 / complex64 GEMMs: TCI_F32_OZAKI_INT8 (default) or TCI_F32_FP64_CORES
  void *dev_scratch;    // reductions (vec.cu): allocated once at creation
  void *host_scratch;   // pinned, reduction results
  cudaStream_t copy_stream;   // library-owned (created on first use): staged H2D / D2H copies
  // peer-memory all-gather (tci_gather_register): P pointers of each kind
  int g_nranks, g_rank;
  void *g_full[8], *g_flags[8];
  uint32_t g_epoch;
  int *g_err;                 // device: set when a barrier timed out
  cudaEvent_t evs[8];         // ordering events between the context and copy streams
  cudaStream_t d2h_stream;    // library-owned lane 2 (tci_copy_async), created on first use
  cudaEvent_t lane_ev[16];    // tci_lane_record / tci_lane_wait slots
  // Ozaki accuracy guard (R26): tolerance on the estimated relative
  // Frobenius error (<= 0: off) and device-resident statistics
  double oz_tol;
  tci::OzGuard *oz_guard;
  int oz_gauss;         // complex Ozaki variant: 1 Gaussian moduli (R33), 0 3M
  bool capturing;       // between tci_graph_begin and tci_graph_end
  int svd_last_sweeps;  // Jacobi sweeps of the last svd / trunc_svd (tci_svd_info)
  double svd_last_off;  // its final off-diagonal measure
};

struct tci_graph_s {
  uint32_t magic;
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  int64_t kernels;      // kernels recorded (added to the context's launch count per replay)
};

struct tci_tensor_s {
  uint32_t magic;
  tci_ctx_s *ctx;
  tci_dtype_t dtype;
  int order;
  int64_t shape[TCI_MAX_ORDER];
  void *data;
  bool host;
};

namespace tci {

constexpr uint32_t kCtxMagic = 0x7c1c7c1cu;
constexpr uint32_t kTenMagic = 0x7e4507e4u;

// thread-local error message
void set_error(const char *fmt, ...);
const char *last_error();

#define TCI_FAIL(code, ...)        \
  do {                             \
    ::tci::set_error(__VA_ARGS__); \
    return (code);                 \
  } while (0)

#define TCI_CUDA_CHECK(expr)                                                                  \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      TCI_FAIL(TCI_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

// A dense row-major view (the data of a descriptor).
struct View {
  tci_dtype_t dtype;
  int order;
  int64_t shape[kMaxOrder];
  void *data;
  int64_t size() const {
    int64_t n = 1;
    for (int i = 0; i < order; i++) n *= shape[i];
    return n;
  }
  size_t bytes() const { return (size_t)size() * dtype_size(dtype); }
};

inline View view_of(const tci_tensor_s *t) {
  View v;
  v.dtype = t->dtype;
  v.order = t->order;
  for (int i = 0; i < t->order; i++) v.shape[i] = t->shape[i];
  v.data = t->data;
  return v;
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Label validation + output shape, identical check order to the oracle
// (DESIGN.md "Error kinds").
tci_status_t contract_shape(int na, const int64_t *sa, const int32_t *la, int nb, const int64_t *sb,
                            const int32_t *lb, int nc, const int32_t *lc, int64_t *sc);

// Plan + (unless dry_run) execute a pairwise contraction on ctx->stream using
// scratch [ws, ws + ws_bytes). *ws_needed receives the scratch requirement.
tci_status_t contract_exec(tci_ctx_s *ctx, const View &a, const int32_t *la, const View &b,
                           const int32_t *lb, const View &c, const int32_t *lc, bool dry_run,
                           size_t *ws_needed, void *ws, size_t ws_bytes);

// Permute a dense view: out bond k = in bond perm[k]. out must not overlap in.
tci_status_t permute_exec(tci_ctx_s *ctx, const View &in, const int32_t *perm, void *out_data);

// Launch wrappers: count launches and (when profiling) bracket each kernel
// with CUDA events on ctx->stream, recording its algorithmic flops / bytes.
enum { kProfGemm = 0, kProfSkinny = 1, kProfPermute = 2, kProfI8 = 3 };
tci_status_t run_gemm(tci_ctx_s *ctx, const GemmProblem &g);
tci_status_t run_skinny(tci_ctx_s *ctx, const SkinnyProblem &p);
tci_status_t run_permute(tci_ctx_s *ctx, const PermuteProblem &p);
tci_status_t run_tebd(tci_ctx_s *ctx, const TebdProblem &t);

// Vector ops and Lanczos (lanczos.cpp)
tci_status_t vec_norm(tci_ctx_s *ctx, const View &a, double *nrm);
tci_status_t vec_inner(tci_ctx_s *ctx, const View &a, const View &b, int conj_a, double out[2]);
tci_status_t vec_lincomb(tci_ctx_s *ctx, int m, const View *ins, const double *coefs, const View &out);
tci_status_t lanczos_bytes(tci_ctx_s *ctx, const View &L, const View &W1, const View &W2, const View &R,
                           const View &psi, int max_iter, size_t *bytes, size_t *heff_b);
tci_status_t lanczos_exec(tci_ctx_s *ctx, const View &L, const View &W1, const View &W2, const View &R,
                          const View &psi, int max_iter, double tol, double *energy, int *iters);
typedef int (*ag_fn)(const void *, void *, size_t, int, void *, cudaStream_t);
ag_fn nccl_allgather_ptr();

// Chains (chains.cpp)
tci_status_t heff_plan_bytes(tci_dtype_t dt, int64_t chi_l, int64_t chi_lo, int64_t chi_r,
                             int64_t chi_ro, int64_t d, int64_t D, int64_t D1, int64_t D2,
                             size_t *bytes, bool *fused_w12, int zalgo = 0);
// Host staging for tci_heff_apply_staged: ev_in / ev_R are recorded on the
// copy stream after the H2D copies of (L, W1, W2, psi) / R; GEMM1 waits for
// ev_in, GEMM4 for ev_R, and every finished row chunk of out is copied to
// out_host on the copy stream.
struct HeffStaging {
  tci_ctx_s *ctx;
  cudaEvent_t ev_in, ev_R, ev_rows, ev_L;
  // L streamed in column blocks during GEMM1 (L[a, (w b)]: chi_l rows of
  // m_cols elements); R copied after the last block
  const char *L_host;
  char *L_dev;
  int64_t L_rows, L_cols, es;
  const char *R_host;
  char *R_dev;
  size_t R_bytes;
  char *out_host;
  const char *out_dev;
  int64_t row_bytes;
  int64_t chunk_rows;
  cudaError_t err;
};
// Peer-memory all-gather of the output slab (tci_heff_apply_gather): GEMM4's
// epilogue also stores every element at peer_out[p] (same layout); `fused`
// reports whether it did (else the caller pushes the slab after the chain)
struct HeffGather {
  int npeer;
  void *peer_out[7];
  bool fused;
};
tci_status_t heff_exec(tci_ctx_s *ctx, const View &L, const View &W1, const View &W2, const View &R,
                       const View &psi, const View &out, HeffStaging *stage = nullptr,
                       HeffGather *gather = nullptr);
tci_status_t tebd_exec(tci_ctx_s *ctx, const View &A, const char *la, const View &B, const char *lb,
                       const View &U, const char *lu, const View &T, const char *lt, size_t *ws_query = nullptr);

// Environment updates (env.cpp)
tci_status_t env_bytes(tci_ctx_s *ctx, int side, const View &E, const View &K, const View &W, const View &B,
                       const View &O, size_t *bytes);
tci_status_t env_exec(tci_ctx_s *ctx, int side, const View &E, const View &K, const View &W, const View &B,
                      const View &O);

// SVD (svd.cpp)
tci_status_t svd_bytes(tci_dtype_t dt, int order, const int64_t *shape, int k, size_t *bytes);
tci_status_t svd_exec(tci_ctx_s *ctx, const View &a, int k, bool trunc, int64_t chi_min, int64_t chi_max,
                      double target, double s_min, tci_tensor_s *tu, tci_tensor_s *ts, tci_tensor_s *tv,
                      double *trunc_err, int64_t *chi_out, void *ws = nullptr, size_t ws_bytes = 0);

// Zip-up MPS-MPO application with truncation (zipup.cpp)
tci_status_t zipup_bytes(tci_ctx_s *ctx, int n, const tci_tensor_s *const *A, const tci_tensor_s *const *W,
                         int64_t chi_max, size_t *bytes);
tci_status_t zipup_exec(tci_ctx_s *ctx, int n, const tci_tensor_s *const *A, const tci_tensor_s *const *W,
                        tci_tensor_s *const *B, int64_t chi_max, double s_min, double *trunc_err);

}  // namespace tci
