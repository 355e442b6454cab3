// abi.cpp -- the extern "C" entry points of libtci_b200 (include/tci_b200.h):
// context lifecycle, descriptors and queries,
// reshape, transpose, contract,
// chains, NCCL all-gather, TCI_VERBOSE diagnostics.
// Every call validates all arguments before enqueueing any kernel.
#include <dlfcn.h>
#include <map>
#include <mutex>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "runtime.h"

namespace tci {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}
const char *last_error() { return g_err; }

namespace {
struct ProfScope {
  tci_ctx_s *ctx;
  int kind;
  double flops, bytes;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(tci_ctx_s *c, int k, double f, double by) : ctx(c), kind(k), flops(f), bytes(by) {
    if (!ctx->prof_on) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, ctx->stream);
  }
  void done() {
    if (!ctx->prof_on || !a) return;
    cudaEventRecord(b, ctx->stream);
    ctx->prof.push_back({kind, a, b, flops, bytes});
    a = b = nullptr;
  }
};
}  // namespace

tci_status_t run_gemm(tci_ctx_s *ctx, const GemmProblem &g) {
  const bool cplx = dtype_is_complex(g.dtype);
  const double es = (double)dtype_size(g.dtype);
  ProfScope ps(ctx, kProfGemm, (cplx ? 8.0 : 2.0) * g.M * g.N * g.K,
               es * ((double)g.M * g.K + (double)g.K * g.N + (double)g.M * g.N));
  OzProf pf{};
  GemmProblem gg = g;
  if (ctx->prof_on && g.zalgo == kZOzaki) gg.oz_prof = &pf;
  const bool f32 = g.dtype == TCI_R32 || g.dtype == TCI_C64;
  gg.oz_tol = (f32 && ctx->oz_tol > 0.0) ? std::max(ctx->oz_tol, kOzakiF32Tol) : ctx->oz_tol;
  gg.oz_guard = ctx->oz_guard;
  gg.oz_gauss = ctx->oz_gauss;
  TCI_CUDA_CHECK(launch_gemm(gg, ctx->stream, &ctx->launches));
  ps.done();
  for (int i = 0; i < pf.n; i++) ctx->prof.push_back({kProfI8, pf.a[i], pf.b[i], pf.ops[i], 0.0});
  return TCI_OK;
}

tci_status_t run_skinny(tci_ctx_s *ctx, const SkinnyProblem &p) {
  const bool cplx = dtype_is_complex(p.dtype);
  const double nb = (double)p.nb[0] * p.nb[1] * p.nb[2];
  ProfScope ps(ctx, kProfSkinny, (cplx ? 8.0 : 2.0) * nb * p.K * p.N,
               (double)dtype_size(p.dtype) * nb * (p.K + p.N));
  TCI_CUDA_CHECK(launch_skinny(p, ctx->stream, &ctx->launches));
  ps.done();
  return TCI_OK;
}

tci_status_t run_tebd(tci_ctx_s *ctx, const TebdProblem &t) {
  const double M = 2.0 * t.chi_a, N = 2.0 * t.chi_c, K = (double)t.chi_b;
  ProfScope ps(ctx, kProfGemm, 2.0 * M * N * K + 2.0 * 16.0 * t.chi_a * t.chi_c,
               8.0 * (M * K + K * N + M * N));
  // TMA-loaded tiles (tebd_tma.cu) unless TCI_TEBD_TMA=0; the cp.async kernel otherwise
  static const bool use_tma = [] {
    const char *e = getenv("TCI_TEBD_TMA");
    return !(e && !strcmp(e, "0"));
  }();
  if (use_tma && tebd_tma_supported(t))
    TCI_CUDA_CHECK(launch_tebd_tma(t, ctx->stream, &ctx->launches));
  else
    TCI_CUDA_CHECK(launch_tebd_fused(t, ctx->stream, &ctx->launches));
  ps.done();
  return TCI_OK;
}

tci_status_t run_permute(tci_ctx_s *ctx, const PermuteProblem &p) {
  ProfScope ps(ctx, kProfPermute, 0.0, 2.0 * (double)p.total * (double)p.esize);
  TCI_CUDA_CHECK(launch_permute(p, ctx->stream, &ctx->launches));
  ps.done();
  return TCI_OK;
}

}  // namespace tci

using namespace tci;

namespace {

tci_status_t check_ctx(tci_ctx_t ctx) {
  if (!ctx) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL context");
  if (ctx->magic != kCtxMagic) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "not a context handle");
  if (!ctx->alive) TCI_FAIL(TCI_ERR_DEAD_CONTEXT, "context was destroyed (P:356, P:2367-2373)");
  return TCI_OK;
}

tci_status_t check_ten(tci_ctx_t ctx, tci_tensor_t t, bool need_device) {
  if (!t) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL tensor");
  if (t->magic != kTenMagic) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "not a tensor descriptor");
  if (t->ctx != ctx) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "tensor belongs to another context");
  if (need_device && t->host)
    TCI_FAIL(TCI_ERR_UNSUPPORTED, "compute calls need device memory (use tci_copy for host data)");
  return TCI_OK;
}

#define CHECK(x)                   \
  do {                             \
    tci_status_t _s = (x);         \
    if (_s != TCI_OK) return _s;   \
  } while (0)

const char *dtype_name(tci_dtype_t t) {
  switch (t) {
    case TCI_R32: return "r32";
    case TCI_R64: return "r64";
    case TCI_C64: return "c64";
    case TCI_C128: return "c128";
  }
  return "?";
}

// TCI_VERBOSE: one line per call; level 2 adds time_us
struct Verbose {
  tci_ctx_t ctx;
  const char *op;
  std::string shapes;
  tci_dtype_t dt;
  std::chrono::steady_clock::time_point t0;
  Verbose(tci_ctx_t c, const char *o, std::initializer_list<tci_tensor_t> ts) : ctx(c), op(o) {
    if (!ctx || ctx->verbose <= 0) return;
    dt = TCI_R64;
    bool first = true;
    for (tci_tensor_t t : ts) {
      if (!t) continue;
      if (!first) shapes += ';';
      first = false;
      dt = t->dtype;
      for (int k = 0; k < t->order; k++) {
        if (k) shapes += ',';
        shapes += std::to_string(t->shape[k]);
      }
    }
    if (ctx->verbose >= 2) {
      cudaStreamSynchronize(ctx->stream);
      t0 = std::chrono::steady_clock::now();
    }
  }
  ~Verbose() {
    if (!ctx || ctx->verbose <= 0) return;
    if (ctx->verbose >= 2) {
      cudaStreamSynchronize(ctx->stream);
      const auto us = std::chrono::duration_cast<std::chrono::microseconds>(
                          std::chrono::steady_clock::now() - t0)
                          .count();
      fprintf(stderr, "tci:%s shapes=[%s] dtype=%s time_us=%lld\n", op, shapes.c_str(),
              dtype_name(dt), (long long)us);
    } else {
      fprintf(stderr, "tci:%s shapes=[%s] dtype=%s\n", op, shapes.c_str(), dtype_name(dt));
    }
  }
};

int read_verbose() {
  const char *v = getenv("TCI_VERBOSE");
  if (!v || !*v) return 0;
  char *end = nullptr;
  long x = strtol(v, &end, 10);
  if (*end || x < 0) {
    fprintf(stderr, "tci: warning: TCI_VERBOSE=%s is not 0, 1 or 2; using 0\n", v);
    return 0;
  }
  return x > 2 ? 2 : (int)x;
}

tci_status_t parse_labels(const char *s, int order, int32_t *out, const char *what) {
  if (!s) TCI_FAIL(TCI_ERR_PARSE, "%s: NULL label string", what);
  const size_t n = strnlen(s, kMaxOrder + 1);
  if ((int)n != order)
    TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "%s: label string \"%s\" has %zu labels for order %d", what, s, n, order);
  for (int i = 0; i < order; i++) out[i] = (unsigned char)s[i];
  return TCI_OK;
}

}  // namespace

extern "C" {

const char *tci_version(void) { return "1.0"; }

const char *tci_last_error(void) { return tci::last_error(); }

tci_status_t tci_create_context(tci_ctx_t *ctx, int device, void *stream) {
  if (!ctx) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "ctx out-pointer is NULL");
  int n = 0;
  TCI_CUDA_CHECK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "device %d of %d", device, n);
  TCI_CUDA_CHECK(cudaSetDevice(device));
  tci_ctx_s *c = new tci_ctx_s();
  c->magic = kCtxMagic;
  c->alive = true;
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  c->verbose = read_verbose();
  c->ws = nullptr;
  c->ws_bytes = 0;
  c->launches = 0;
  c->nccl_comm = nullptr;
  c->nranks = 1;
  c->rank = 0;
  c->plan_hits = c->plan_misses = 0;
  c->prof_on = false;
  c->zgemm_algo = kZ3M;
  if (const char *e = getenv("TCI_ZGEMM_ALGO")) {
    if (!strcmp(e, "4m") || !strcmp(e, "4M")) c->zgemm_algo = kZ4M;
    else if (!strcmp(e, "ozaki") || !strcmp(e, "OZAKI")) c->zgemm_algo = kZOzaki;
  }
  c->dev_scratch = nullptr;
  c->host_scratch = nullptr;
  c->copy_stream = nullptr;
  for (auto &e : c->evs) e = nullptr;
  c->d2h_stream = nullptr;
  for (auto &e : c->lane_ev) e = nullptr;
  c->g_nranks = 1;
  c->g_rank = 0;
  for (int i = 0; i < 8; i++) c->g_full[i] = c->g_flags[i] = nullptr;
  c->g_epoch = 0;
  c->g_err = nullptr;
  c->capturing = false;
  c->svd_last_sweeps = 0;
  c->svd_last_off = 0.0;
  c->oz_tol = kOzakiDefaultTol;
  if (const char *e = getenv("TCI_OZAKI_GUARD")) {
    if (!strcmp(e, "0") || !strcmp(e, "off")) c->oz_tol = 0.0;
  }
  c->oz_guard = nullptr;
  c->oz_gauss = 1;
  c->f32_algo = TCI_F32_OZAKI_INT8;
  if (const char *e = getenv("TCI_F32_ALGO")) {
    if (!strcmp(e, "fp64") || !strcmp(e, "simt")) c->f32_algo = TCI_F32_FP64_CORES;
  }
  if (const char *e = getenv("TCI_OZAKI_CPLX")) {
    if (!strcmp(e, "3m") || !strcmp(e, "3M")) c->oz_gauss = 0;
  }
  {
    cudaError_t e1 = cudaMalloc(&c->dev_scratch, reduce_scratch_bytes());
    cudaError_t e2 = cudaMallocHost(&c->host_scratch, 2 * kMaxMIOut * sizeof(double) + 64);
    cudaError_t e3 = cudaMalloc(&c->oz_guard, sizeof(OzGuard));
    if (e3 == cudaSuccess) e3 = cudaMemset(c->oz_guard, 0, sizeof(OzGuard));
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      if (c->dev_scratch) cudaFree(c->dev_scratch);
      if (c->host_scratch) cudaFreeHost(c->host_scratch);
      if (c->oz_guard) cudaFree(c->oz_guard);
      delete c;
      TCI_FAIL(TCI_ERR_CUDA, "context scratch allocation failed");
    }
  }
  *ctx = c;
  return TCI_OK;
}

// NCCL through dlopen of the process's libnccl.so.2 (torch ships it); the
// minimal ABI used here is stable across NCCL 2.x.
typedef struct { char internal[128]; } nccl_uid_t;
typedef int (*nccl_get_uid_fn)(nccl_uid_t *);
typedef int (*nccl_init_rank_fn)(void **, int, nccl_uid_t, int);
typedef int (*nccl_allgather_fn)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*nccl_destroy_fn)(void *);
typedef const char *(*nccl_errstr_fn)(int);
static struct {
  void *h = nullptr;
  nccl_get_uid_fn get_uid;
  nccl_init_rank_fn init_rank;
  nccl_allgather_fn allgather;
  nccl_destroy_fn destroy;
  nccl_errstr_fn errstr;
} g_nccl;

static tci_status_t nccl_load() {
  if (g_nccl.h) return TCI_OK;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW);
  if (!h) TCI_FAIL(TCI_ERR_NCCL, "cannot load libnccl.so.2: %s", dlerror());
  g_nccl.get_uid = (nccl_get_uid_fn)dlsym(h, "ncclGetUniqueId");
  g_nccl.init_rank = (nccl_init_rank_fn)dlsym(h, "ncclCommInitRank");
  g_nccl.allgather = (nccl_allgather_fn)dlsym(h, "ncclAllGather");
  g_nccl.destroy = (nccl_destroy_fn)dlsym(h, "ncclCommDestroy");
  g_nccl.errstr = (nccl_errstr_fn)dlsym(h, "ncclGetErrorString");
  if (!g_nccl.get_uid || !g_nccl.init_rank || !g_nccl.allgather || !g_nccl.destroy)
    TCI_FAIL(TCI_ERR_NCCL, "libnccl.so.2 lacks a required symbol");
  g_nccl.h = h;
  return TCI_OK;
}

static void prof_clear(tci_ctx_t ctx);

tci_status_t tci_destroy_context(tci_ctx_t ctx) {
  CHECK(check_ctx(ctx));
  Verbose vb(ctx, "destroy_context", {});
  if (ctx->nccl_comm && g_nccl.destroy) g_nccl.destroy(ctx->nccl_comm);
  cudaStreamSynchronize(ctx->stream);
  prof_clear(ctx);
  ctx->prof_on = false;
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
    ctx->copy_stream = nullptr;
  }
  for (auto &e : ctx->evs)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  if (ctx->d2h_stream) {
    cudaStreamSynchronize(ctx->d2h_stream);
    cudaStreamDestroy(ctx->d2h_stream);
    ctx->d2h_stream = nullptr;
  }
  for (auto &e : ctx->lane_ev)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  if (ctx->dev_scratch) cudaFree(ctx->dev_scratch);
  if (ctx->host_scratch) cudaFreeHost(ctx->host_scratch);
  if (ctx->oz_guard) cudaFree(ctx->oz_guard);
  ctx->oz_guard = nullptr;
  if (ctx->g_err) cudaFree(ctx->g_err);
  ctx->g_err = nullptr;
  ctx->g_nranks = 1;
  ctx->dev_scratch = ctx->host_scratch = nullptr;
  ctx->nccl_comm = nullptr;
  ctx->plan_cache.clear();
  ctx->ws = nullptr;
  ctx->ws_bytes = 0;
  ctx->alive = false;   // handle kept (not freed) so later calls see DEAD_CONTEXT
  return TCI_OK;
}

// ---- CUDA-graph capture (host-path latency of short chains) ----
namespace {
constexpr uint32_t kGraphMagic = 0x54434947u;   // "TCIG"
int64_t g_capture_launch0[64];
}  // namespace

tci_status_t tci_graph_begin(tci_ctx_t ctx) {
  CHECK(check_ctx(ctx));
  if (ctx->capturing) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "graph capture already active on this context");
  if (ctx->stream == nullptr || ctx->stream == cudaStreamLegacy)
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "the legacy NULL stream cannot be captured; create the context on a stream");
  TCI_CUDA_CHECK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  ctx->capturing = true;
  g_capture_launch0[ctx->device & 63] = ctx->launches;
  return TCI_OK;
}

tci_status_t tci_graph_end(tci_ctx_t ctx, tci_graph_t *graph) {
  CHECK(check_ctx(ctx));
  if (!ctx->capturing) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "no graph capture active on this context");
  ctx->capturing = false;
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);   // always ends the capture
  if (e != cudaSuccess || !g) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    TCI_FAIL(TCI_ERR_CUDA, "graph capture failed: %s (a call in the capture synchronized or read results)",
             cudaGetErrorString(e));
  }
  if (!graph) {
    cudaGraphDestroy(g);
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL graph out-pointer");
  }
  cudaGraphExec_t x = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&x, g, 0);
  if (ei != cudaSuccess) {
    cudaGraphDestroy(g);
    TCI_FAIL(TCI_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ei));
  }
  auto *h = new tci_graph_s{kGraphMagic, g, x, ctx->launches - g_capture_launch0[ctx->device & 63]};
  ctx->launches = g_capture_launch0[ctx->device & 63];   // nothing ran yet
  *graph = h;
  return TCI_OK;
}

tci_status_t tci_graph_launch(tci_ctx_t ctx, tci_graph_t graph) {
  CHECK(check_ctx(ctx));
  if (!graph || graph->magic != kGraphMagic) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "not a graph handle");
  if (ctx->capturing) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "graph launch inside a capture");
  TCI_CUDA_CHECK(cudaGraphLaunch(graph->exec, ctx->stream));
  ctx->launches += graph->kernels;
  return TCI_OK;
}

tci_status_t tci_graph_destroy(tci_graph_t graph) {
  if (!graph || graph->magic != kGraphMagic) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "not a graph handle");
  graph->magic = 0;
  cudaGraphExecDestroy(graph->exec);
  cudaGraphDestroy(graph->graph);
  delete graph;
  return TCI_OK;
}

tci_status_t tci_synchronize(tci_ctx_t ctx) {
  CHECK(check_ctx(ctx));
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return TCI_OK;
}

tci_status_t tci_workspace_attach(tci_ctx_t ctx, void *dev_ws, size_t bytes) {
  CHECK(check_ctx(ctx));
  if (dev_ws && ((uintptr_t)dev_ws % 256))
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  ctx->ws = bytes ? dev_ws : nullptr;
  ctx->ws_bytes = dev_ws ? bytes : 0;
  return TCI_OK;
}

tci_status_t tci_set_gemm_algorithm(tci_ctx_t ctx, int algo) {
  CHECK(check_ctx(ctx));
  if (algo != TCI_GEMM_DMMA_3M && algo != TCI_GEMM_DMMA_4M && algo != TCI_GEMM_OZAKI_INT8)
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "unknown GEMM algorithm %d", algo);
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));   // scratch layouts may change
  ctx->zgemm_algo = algo;
  return TCI_OK;
}

tci_status_t tci_set_ozaki_guard(tci_ctx_t ctx, double tol) {
  CHECK(check_ctx(ctx));
  if (!(tol == tol)) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "tolerance is NaN");
  ctx->oz_tol = tol > 0.0 ? tol : 0.0;
  return TCI_OK;
}

tci_status_t tci_set_f32_algorithm(tci_ctx_t ctx, int algo) {
  CHECK(check_ctx(ctx));
  if (algo != TCI_F32_OZAKI_INT8 && algo != TCI_F32_FP64_CORES)
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "unknown float32 GEMM algorithm %d", algo);
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  ctx->f32_algo = algo;
  return TCI_OK;
}

tci_status_t tci_set_ozaki_complex(tci_ctx_t ctx, int variant) {
  CHECK(check_ctx(ctx));
  if (variant != TCI_OZAKI_CPLX_GAUSS && variant != TCI_OZAKI_CPLX_3M)
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "unknown Ozaki complex variant %d", variant);
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  ctx->oz_gauss = variant == TCI_OZAKI_CPLX_GAUSS ? 1 : 0;
  return TCI_OK;
}

tci_status_t tci_ozaki_guard_stats(tci_ctx_t ctx, int reset, int64_t *gemms, int64_t *fallbacks, int64_t *balanced,
                                   double *last_est, double *max_est) {
  CHECK(check_ctx(ctx));
  OzGuard h{};
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  TCI_CUDA_CHECK(cudaMemcpy(&h, ctx->oz_guard, sizeof h, cudaMemcpyDeviceToHost));
  if (gemms) *gemms = (int64_t)h.gemms;
  if (fallbacks) *fallbacks = (int64_t)h.fallbacks;
  if (balanced) *balanced = (int64_t)h.balanced;
  if (last_est) *last_est = h.last_est;
  if (max_est) *max_est = h.max_est;
  if (reset) TCI_CUDA_CHECK(cudaMemset(ctx->oz_guard, 0, sizeof(OzGuard)));
  return TCI_OK;
}

tci_status_t tci_get_gemm_algorithm(tci_ctx_t ctx, int *algo) {
  CHECK(check_ctx(ctx));
  if (!algo) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  *algo = ctx->zgemm_algo;
  return TCI_OK;
}

tci_status_t tci_launch_count(tci_ctx_t ctx, int64_t *count) {
  CHECK(check_ctx(ctx));
  if (!count) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL count");
  *count = ctx->launches;
  return TCI_OK;
}

static void prof_clear(tci_ctx_t ctx) {
  for (auto &r : ctx->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  ctx->prof.clear();
}

tci_status_t tci_profile_enable(tci_ctx_t ctx, int on) {
  CHECK(check_ctx(ctx));
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  prof_clear(ctx);
  ctx->prof_on = on != 0;
  return TCI_OK;
}

tci_status_t tci_profile_query(tci_ctx_t ctx, int kind, int64_t *launches, double *ms, double *flops,
                               double *bytes) {
  CHECK(check_ctx(ctx));
  if (kind < 0 || kind > 3) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "profile kind %d", kind);
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  int64_t n = 0;
  double t = 0, f = 0, by = 0;
  for (auto &r : ctx->prof) {
    if (r.kind != kind) continue;
    float x = 0;
    TCI_CUDA_CHECK(cudaEventElapsedTime(&x, r.a, r.b));
    n++;
    t += x;
    f += r.flops;
    by += r.bytes;
  }
  if (launches) *launches = n;
  if (ms) *ms = t;
  if (flops) *flops = f;
  if (bytes) *bytes = by;
  return TCI_OK;
}

tci_status_t tci_tensor_create(tci_ctx_t ctx, tci_dtype_t dtype, int order, const int64_t *shape,
                               void *data, tci_tensor_t *out) {
  CHECK(check_ctx(ctx));
  if (!out) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "out is NULL");
  if (dtype < TCI_R32 || dtype > TCI_C128) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "bad dtype %d", (int)dtype);
  if (order < 0) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "negative order");
  if (order > kMaxOrder) TCI_FAIL(TCI_ERR_UNSUPPORTED, "order %d > %d", order, kMaxOrder);
  if (order > 0 && !shape) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "shape is NULL");
  for (int k = 0; k < order; k++)
    if (shape[k] < 1) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "dimension %d is %lld (< 1, reading R13)", k, (long long)shape[k]);
  if (!data) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "data is NULL");
  const size_t es = dtype_size(dtype);
  if ((uintptr_t)data % (dtype == TCI_C128 ? 16 : (es > 8 ? 8 : es)))
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "data is not aligned for dtype %s", dtype_name(dtype));
  cudaPointerAttributes attr;
  bool host = true;
  if (cudaPointerGetAttributes(&attr, data) == cudaSuccess)
    host = !(attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged);
  cudaGetLastError();   // clear a possible "invalid value" from unregistered host memory
  tci_tensor_s *t = new tci_tensor_s();
  t->magic = kTenMagic;
  t->ctx = ctx;
  t->dtype = dtype;
  t->order = order;
  for (int k = 0; k < order; k++) t->shape[k] = shape[k];
  t->data = data;
  t->host = host;
  *out = t;
  return TCI_OK;
}

tci_status_t tci_tensor_free(tci_ctx_t ctx, tci_tensor_t t) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, t, false));
  t->magic = 0;
  delete t;
  return TCI_OK;
}

tci_status_t tci_order(tci_ctx_t ctx, tci_tensor_t t, int *order) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, t, false));
  if (!order) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  *order = t->order;
  return TCI_OK;
}

tci_status_t tci_shape(tci_ctx_t ctx, tci_tensor_t t, int64_t *shape) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, t, false));
  if (!shape && t->order) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  for (int k = 0; k < t->order; k++) shape[k] = t->shape[k];
  return TCI_OK;
}

tci_status_t tci_size(tci_ctx_t ctx, tci_tensor_t t, int64_t *n) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, t, false));
  if (!n) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  *n = view_of(t).size();
  return TCI_OK;
}

tci_status_t tci_size_bytes(tci_ctx_t ctx, tci_tensor_t t, int64_t *bytes) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, t, false));
  if (!bytes) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  *bytes = (int64_t)view_of(t).bytes();
  return TCI_OK;
}

tci_status_t tci_copy(tci_ctx_t ctx, tci_tensor_t src, tci_tensor_t dst) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, src, false));
  CHECK(check_ten(ctx, dst, false));
  if (src->dtype != dst->dtype) TCI_FAIL(TCI_ERR_UNSUPPORTED, "copy: dtype mismatch");
  if (view_of(src).size() != view_of(dst).size()) TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "copy: element counts differ");
  Verbose vb(ctx, "copy", {src, dst});
  TCI_CUDA_CHECK(cudaMemcpyAsync(dst->data, src->data, view_of(src).bytes(), cudaMemcpyDefault, ctx->stream));
  return TCI_OK;
}

static tci_status_t lane_stream(tci_ctx_t ctx, int lane, cudaStream_t *s) {
  if (lane < 0 || lane > 2) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "lane %d (0 context, 1 h2d, 2 d2h)", lane);
  if (lane == 0) {
    *s = ctx->stream;
    return TCI_OK;
  }
  cudaStream_t &ls = lane == 1 ? ctx->copy_stream : ctx->d2h_stream;
  if (!ls) {
    TCI_CUDA_CHECK(cudaSetDevice(ctx->device));
    TCI_CUDA_CHECK(cudaStreamCreateWithFlags(&ls, cudaStreamNonBlocking));
  }
  *s = ls;
  return TCI_OK;
}

tci_status_t tci_copy_async(tci_ctx_t ctx, tci_tensor_t src, tci_tensor_t dst, int lane) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, src, false));
  CHECK(check_ten(ctx, dst, false));
  if (src->dtype != dst->dtype) TCI_FAIL(TCI_ERR_UNSUPPORTED, "copy: dtype mismatch");
  if (view_of(src).size() != view_of(dst).size()) TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "copy: element counts differ");
  cudaStream_t s;
  CHECK(lane_stream(ctx, lane, &s));
  Verbose vb(ctx, "copy_async", {src, dst});
  TCI_CUDA_CHECK(cudaMemcpyAsync(dst->data, src->data, view_of(src).bytes(), cudaMemcpyDefault, s));
  return TCI_OK;
}

tci_status_t tci_lane_record(tci_ctx_t ctx, int lane, int slot) {
  CHECK(check_ctx(ctx));
  if (slot < 0 || slot >= 16) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "slot %d (0..15)", slot);
  cudaStream_t s;
  CHECK(lane_stream(ctx, lane, &s));
  if (!ctx->lane_ev[slot]) TCI_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->lane_ev[slot], cudaEventDisableTiming));
  TCI_CUDA_CHECK(cudaEventRecord(ctx->lane_ev[slot], s));
  return TCI_OK;
}

tci_status_t tci_lane_wait(tci_ctx_t ctx, int lane, int slot) {
  CHECK(check_ctx(ctx));
  if (slot < 0 || slot >= 16) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "slot %d (0..15)", slot);
  cudaStream_t s;
  CHECK(lane_stream(ctx, lane, &s));
  if (!ctx->lane_ev[slot]) return TCI_OK;   // never recorded: nothing to wait for
  TCI_CUDA_CHECK(cudaStreamWaitEvent(s, ctx->lane_ev[slot], 0));
  return TCI_OK;
}

tci_status_t tci_reshape(tci_ctx_t ctx, tci_tensor_t t, int order, const int64_t *new_shape) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, t, false));
  if (order < 0) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "negative order");
  if (order > kMaxOrder) TCI_FAIL(TCI_ERR_UNSUPPORTED, "order > %d", kMaxOrder);
  if (order && !new_shape) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL shape");
  int64_t n = 1;
  for (int k = 0; k < order; k++) {
    if (new_shape[k] < 1) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "dimension %d < 1", k);
    n *= new_shape[k];
  }
  if (n != view_of(t).size())
    TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "reshape changes the element count (%lld -> %lld)",
             (long long)view_of(t).size(), (long long)n);
  Verbose vb(ctx, "reshape", {t});
  t->order = order;
  for (int k = 0; k < order; k++) t->shape[k] = new_shape[k];
  return TCI_OK;
}

tci_status_t tci_permute(tci_ctx_t ctx, tci_tensor_t in, const int32_t *new_order, tci_tensor_t out) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, in, true));
  CHECK(check_ten(ctx, out, true));
  if (in->order && !new_order) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL new_order");
  if (in->dtype != out->dtype) TCI_FAIL(TCI_ERR_UNSUPPORTED, "permute: dtype mismatch");
  if (in->order != out->order) TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "permute: order mismatch");
  bool seen[kMaxOrder] = {};
  for (int k = 0; k < in->order; k++) {
    if (new_order[k] < 0 || new_order[k] >= in->order || seen[new_order[k]])
      TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "new_order is not a permutation");
    seen[new_order[k]] = true;
  }
  for (int k = 0; k < in->order; k++)
    if (out->shape[k] != in->shape[new_order[k]])
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "permute: out.shape[%d] must be in.shape[%d]", k, new_order[k]);
  const View vi = view_of(in), vo = view_of(out);
  const char *a = (const char *)vi.data, *b = (const char *)vo.data;
  if (a < b + vo.bytes() && b < a + vi.bytes())
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "permute: in and out overlap");
  Verbose vb(ctx, "transpose", {in});
  return permute_exec(ctx, vi, new_order, out->data);
}

tci_status_t tci_contract_out_shape(tci_ctx_t ctx, tci_tensor_t a, const int32_t *la, tci_tensor_t b,
                                    const int32_t *lb, int nc, const int32_t *lc, int64_t *shape_c) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, a, false));
  CHECK(check_ten(ctx, b, false));
  if ((a->order && !la) || (b->order && !lb) || (nc && (!lc || !shape_c)))
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL label array");
  int64_t sc[kMaxOrder];
  CHECK(contract_shape(a->order, a->shape, la, b->order, b->shape, lb, nc, lc, sc));
  for (int k = 0; k < nc; k++) shape_c[k] = sc[k];
  return TCI_OK;
}

static tci_status_t contract_common(tci_ctx_t ctx, tci_tensor_t a, const int32_t *la, tci_tensor_t b,
                                    const int32_t *lb, tci_tensor_t c, const int32_t *lc, bool dry,
                                    size_t *need) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, a, !dry));
  CHECK(check_ten(ctx, b, !dry));
  CHECK(check_ten(ctx, c, !dry));
  if ((a->order && !la) || (b->order && !lb) || (c->order && !lc))
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL label array");
  size_t n = 0;
  if (dry) {
    CHECK(contract_exec(ctx, view_of(a), la, view_of(b), lb, view_of(c), lc, true, &n, nullptr, 0));
    if (need) *need = n;
    return TCI_OK;
  }
  // one planning pass: contract_exec checks the workspace before it launches anything
  Verbose vb(ctx, "contract", {a, b, c});
  return contract_exec(ctx, view_of(a), la, view_of(b), lb, view_of(c), lc, false, &n, ctx->ws,
                       ctx->ws_bytes);
}

tci_status_t tci_contract(tci_ctx_t ctx, tci_tensor_t a, const int32_t *la, tci_tensor_t b,
                          const int32_t *lb, tci_tensor_t c, const int32_t *lc) {
  return contract_common(ctx, a, la, b, lb, c, lc, false, nullptr);
}

tci_status_t tci_contract_str(tci_ctx_t ctx, tci_tensor_t a, const char *la, tci_tensor_t b,
                              const char *lb, tci_tensor_t c, const char *lc) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, a, true));
  CHECK(check_ten(ctx, b, true));
  CHECK(check_ten(ctx, c, true));
  int32_t ia[kMaxOrder], ib[kMaxOrder], ic[kMaxOrder];
  CHECK(parse_labels(la, a->order, ia, "a"));
  CHECK(parse_labels(lb, b->order, ib, "b"));
  CHECK(parse_labels(lc, c->order, ic, "c"));
  return contract_common(ctx, a, ia, b, ib, c, ic, false, nullptr);
}

tci_status_t tci_contract_workspace_size(tci_ctx_t ctx, tci_tensor_t a, const int32_t *la,
                                         tci_tensor_t b, const int32_t *lb, tci_tensor_t c,
                                         const int32_t *lc, size_t *bytes) {
  if (!bytes) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  return contract_common(ctx, a, la, b, lb, c, lc, true, bytes);
}

tci_status_t tci_heff_workspace_size(tci_ctx_t ctx, tci_dtype_t dtype, int64_t chi_l, int64_t chi_lo,
                                     int64_t chi_r, int64_t chi_ro, int64_t d, int64_t D, int64_t D1,
                                     int64_t D2, size_t *bytes) {
  CHECK(check_ctx(ctx));
  if (!bytes) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  return heff_plan_bytes(dtype, chi_l, chi_lo, chi_r, chi_ro, d, D, D1, D2, bytes, nullptr, ctx->zgemm_algo);
}

tci_status_t tci_heff_apply(tci_ctx_t ctx, tci_tensor_t L, tci_tensor_t W1, tci_tensor_t W2,
                            tci_tensor_t R, tci_tensor_t psi, tci_tensor_t out) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {L, W1, W2, R, psi, out}) CHECK(check_ten(ctx, t, true));
  const View vo = view_of(out);
  for (tci_tensor_t t : {L, W1, W2, R, psi}) {
    const View v = view_of(t);
    const char *x = (const char *)v.data, *y = (const char *)vo.data;
    if (x < y + vo.bytes() && y < x + v.bytes())
      TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "heff: out overlaps an input");
  }
  Verbose vb(ctx, "heff_apply", {L, W1, W2, R, psi});
  return heff_exec(ctx, view_of(L), view_of(W1), view_of(W2), view_of(R), view_of(psi), vo);
}

tci_status_t tci_heff_apply_staged(tci_ctx_t ctx, tci_tensor_t L_h, tci_tensor_t W1_h, tci_tensor_t W2_h,
                                   tci_tensor_t R_h, tci_tensor_t psi_h, tci_tensor_t out_h, tci_tensor_t L,
                                   tci_tensor_t W1, tci_tensor_t W2, tci_tensor_t R, tci_tensor_t psi,
                                   tci_tensor_t out) {
  CHECK(check_ctx(ctx));
  const tci_tensor_t hs[6] = {L_h, W1_h, W2_h, R_h, psi_h, out_h}, ds[6] = {L, W1, W2, R, psi, out};
  for (int i = 0; i < 6; i++) {
    if (i == 5 && !out_h) {   // inputs staged only: the result stays on the device
      CHECK(check_ten(ctx, ds[i], true));
      continue;
    }
    CHECK(check_ten(ctx, hs[i], false));
    CHECK(check_ten(ctx, ds[i], true));
    if (hs[i]->dtype != ds[i]->dtype || hs[i]->order != ds[i]->order)
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "heff_staged: host / device tensor %d differ in dtype or order", i);
    for (int k = 0; k < ds[i]->order; k++)
      if (hs[i]->shape[k] != ds[i]->shape[k])
        TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "heff_staged: host / device tensor %d differ in shape", i);
  }
  const View vo = view_of(out);
  for (int i = 0; i < 5; i++) {
    const View v = view_of(ds[i]);
    const char *x = (const char *)v.data, *y = (const char *)vo.data;
    if (x < y + vo.bytes() && y < x + v.bytes()) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "heff: out overlaps an input");
  }
  Verbose vb(ctx, "heff_apply_staged", {L, W1, W2, R, psi});
  if (L->order != 3 || R->order != 3) TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "heff: L and R must be order 3");
  if (!ctx->copy_stream) TCI_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  for (auto &e : ctx->evs)
    if (!e) TCI_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaStream_t s0 = ctx->stream, s1 = ctx->copy_stream;
  // the copy stream starts after everything already queued on the context
  // stream -- unless the host output is NULL: then the caller orders the copy
  // lane (tci_lane_wait on lane 1) so a stream of applies can stage step i+1's
  // inputs while step i computes
  if (out_h) {
    TCI_CUDA_CHECK(cudaEventRecord(ctx->evs[0], s0));
    TCI_CUDA_CHECK(cudaStreamWaitEvent(s1, ctx->evs[0], 0));
  }
  auto h2d = [&](int i) -> tci_status_t {
    const View v = view_of(ds[i]);
    TCI_CUDA_CHECK(cudaMemcpyAsync(v.data, hs[i]->data, v.bytes(), cudaMemcpyDefault, s1));
    return TCI_OK;
  };
  // psi and the MPO first (GEMM1's B operand and the MPO pass); L follows in
  // column blocks as GEMM1 reaches them, then R (heff_exec enqueues both)
  for (int i : {4, 1, 2}) CHECK(h2d(i));
  TCI_CUDA_CHECK(cudaEventRecord(ctx->evs[1], s1));
  HeffStaging st{};
  st.ctx = ctx;
  st.ev_in = ctx->evs[1];
  st.ev_R = ctx->evs[2];
  st.ev_rows = ctx->evs[3];
  st.ev_L = ctx->evs[5];
  st.L_host = static_cast<const char *>(L_h->data);
  st.L_dev = static_cast<char *>(L->data);
  st.L_rows = L->shape[0];
  st.L_cols = L->shape[1] * L->shape[2];
  st.es = (int64_t)dtype_size(L->dtype);
  st.R_host = static_cast<const char *>(R_h->data);
  st.R_dev = static_cast<char *>(R->data);
  st.R_bytes = view_of(R).bytes();
  st.out_host = out_h ? static_cast<char *>(out_h->data) : nullptr;
  st.out_dev = static_cast<const char *>(out->data);
  st.row_bytes = out->shape[3] * (int64_t)dtype_size(out->dtype);
  const int64_t rows = out->shape[0] * out->shape[1] * out->shape[2];
  st.chunk_rows = std::max<int64_t>(256, (rows + 7) / 8);
  st.err = cudaSuccess;
  tci_status_t r = heff_exec(ctx, view_of(L), view_of(W1), view_of(W2), view_of(R), view_of(psi), vo, &st);
  // the context stream resumes after the last chunk has reached the host
  TCI_CUDA_CHECK(cudaEventRecord(ctx->evs[4], s1));
  TCI_CUDA_CHECK(cudaStreamWaitEvent(s0, ctx->evs[4], 0));
  return r;
}

tci_status_t tci_env_workspace_size(tci_ctx_t ctx, int side, tci_tensor_t E, tci_tensor_t ket, tci_tensor_t W,
                                    tci_tensor_t bra, tci_tensor_t out, size_t *bytes) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {E, ket, W, bra, out}) CHECK(check_ten(ctx, t, false));
  if (!bytes) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  return env_bytes(ctx, side, view_of(E), view_of(ket), view_of(W), view_of(bra), view_of(out), bytes);
}

tci_status_t tci_env_update(tci_ctx_t ctx, int side, tci_tensor_t E, tci_tensor_t ket, tci_tensor_t W,
                            tci_tensor_t bra, tci_tensor_t out) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {E, ket, W, bra, out}) CHECK(check_ten(ctx, t, true));
  const View vo = view_of(out);
  for (tci_tensor_t t : {E, ket, W, bra}) {
    const View v = view_of(t);
    const char *x = (const char *)v.data, *y = (const char *)vo.data;
    if (x < y + vo.bytes() && y < x + v.bytes())
      TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "env: out overlaps an input");
  }
  Verbose vb(ctx, side == 0 ? "env_update_left" : "env_update_right", {E, ket, W, bra});
  return env_exec(ctx, side, view_of(E), view_of(ket), view_of(W), view_of(bra), vo);
}

tci_status_t tci_cplx_conj(tci_ctx_t ctx, tci_tensor_t in, tci_tensor_t out) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, in, true));
  CHECK(check_ten(ctx, out, true));
  if (in->dtype != out->dtype) TCI_FAIL(TCI_ERR_UNSUPPORTED, "cplx_conj: in and out dtypes differ");
  if (in->order != out->order) TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "cplx_conj: order mismatch");
  for (int k = 0; k < in->order; k++)
    if (in->shape[k] != out->shape[k]) TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "cplx_conj: shapes must be identical");
  const View vi = view_of(in), vo = view_of(out);
  if (vi.data != vo.data) {
    const char *x = (const char *)vi.data, *y = (const char *)vo.data;
    if (x < y + vo.bytes() && y < x + vi.bytes())
      TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "cplx_conj: out partially overlaps in (only in == out is allowed)");
  }
  Verbose vb(ctx, "cplx_conj", {in});
  if (in->dtype == TCI_C128 || in->dtype == TCI_C64) {
    if (in->dtype == TCI_C64) TCI_FAIL(TCI_ERR_UNSUPPORTED, "cplx_conj: complex64 not supported (use complex128)");
    int64_t n = 1;
    for (int k = 0; k < in->order; k++) n *= in->shape[k];
    TCI_CUDA_CHECK(launch_conj(vi.data, vo.data, n, ctx->stream, &ctx->launches));
    return TCI_OK;
  }
  // real element type: (1) in place is a no-op, (2) is a deep copy
  if (vi.data == vo.data) return TCI_OK;
  TCI_CUDA_CHECK(launch_copy(vo.data, vi.data, vi.bytes(), ctx->stream, &ctx->launches));
  return TCI_OK;
}

tci_status_t tci_svd_workspace_size(tci_ctx_t ctx, tci_dtype_t dtype, int order, const int64_t *shape,
                                    int num_of_bds_as_row, size_t *bytes) {
  CHECK(check_ctx(ctx));
  if (!shape || !bytes) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL shape or out");
  if (order < 0 || order > kMaxOrder) TCI_FAIL(TCI_ERR_UNSUPPORTED, "order %d > %d", order, kMaxOrder);
  return svd_bytes(dtype, order, shape, num_of_bds_as_row, bytes);
}

static tci_status_t svd_common(tci_ctx_t ctx, tci_tensor_t a, int k, tci_tensor_t u, tci_tensor_t s,
                               tci_tensor_t v, bool trunc, double *err, int64_t chi_min, int64_t chi_max,
                               double target, double s_min, int64_t *chi_out) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {a, u, s, v}) CHECK(check_ten(ctx, t, true));
  Verbose vb(ctx, trunc ? "trunc_svd" : "svd", {a});
  return svd_exec(ctx, view_of(a), k, trunc, chi_min, chi_max, target, s_min, u, s, v, err, chi_out);
}

tci_status_t tci_svd(tci_ctx_t ctx, tci_tensor_t a, int num_of_bds_as_row, tci_tensor_t u, tci_tensor_t s_diag,
                     tci_tensor_t v_dag) {
  return svd_common(ctx, a, num_of_bds_as_row, u, s_diag, v_dag, false, nullptr, 0, 0, 0.0, 0.0, nullptr);
}

tci_status_t tci_trunc_svd(tci_ctx_t ctx, tci_tensor_t a, int num_of_bds_as_row, tci_tensor_t u,
                           tci_tensor_t s_diag, tci_tensor_t v_dag, double *trunc_err, int64_t chi_min,
                           int64_t chi_max, double target_trunc_err, double s_min, int64_t *chi_out) {
  if (!trunc_err) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "trunc_svd: NULL trunc_err");
  return svd_common(ctx, a, num_of_bds_as_row, u, s_diag, v_dag, true, trunc_err, chi_min, chi_max,
                    target_trunc_err, s_min, chi_out);
}

tci_status_t tci_mps_mpo_zipup_workspace_size(tci_ctx_t ctx, int n, const tci_tensor_t *A, const tci_tensor_t *W,
                                              int64_t chi_max, size_t *bytes) {
  CHECK(check_ctx(ctx));
  if (!A || !W || !bytes) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL argument");
  if (n < 1 || n > 4096) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "zipup: %d sites", n);
  for (int i = 0; i < n; i++) {
    CHECK(check_ten(ctx, A[i], false));
    CHECK(check_ten(ctx, W[i], false));
  }
  return zipup_bytes(ctx, n, A, W, chi_max, bytes);
}

tci_status_t tci_mps_mpo_zipup(tci_ctx_t ctx, int n, const tci_tensor_t *A, const tci_tensor_t *W, tci_tensor_t *B,
                               int64_t chi_max, double s_min, double *trunc_err) {
  CHECK(check_ctx(ctx));
  if (!A || !W || !B) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL site arrays");
  if (n < 1 || n > 4096) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "zipup: %d sites", n);
  for (int i = 0; i < n; i++) {
    CHECK(check_ten(ctx, A[i], true));
    CHECK(check_ten(ctx, W[i], true));
    CHECK(check_ten(ctx, B[i], true));
  }
  Verbose vb(ctx, "mps_mpo_zipup", {A[0], W[0]});
  return zipup_exec(ctx, n, A, W, B, chi_max, s_min, trunc_err);
}

tci_status_t tci_svd_info(tci_ctx_t ctx, int *sweeps, double *off) {
  CHECK(check_ctx(ctx));
  if (sweeps) *sweeps = ctx->svd_last_sweeps;
  if (off) *off = ctx->svd_last_off;
  return TCI_OK;
}

tci_status_t tci_tebd_theta(tci_ctx_t ctx, tci_tensor_t A, const char *la, tci_tensor_t B,
                            const char *lb, tci_tensor_t U, const char *lu, tci_tensor_t theta,
                            const char *lt) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {A, B, U, theta}) CHECK(check_ten(ctx, t, true));
  if (!la || !lb || !lu || !lt) TCI_FAIL(TCI_ERR_PARSE, "tebd: NULL label string");
  Verbose vb(ctx, "tebd_theta", {A, B, U});
  return tebd_exec(ctx, view_of(A), la, view_of(B), lb, view_of(U), lu, view_of(theta), lt);
}

tci_status_t tci_tebd_workspace_size(tci_ctx_t ctx, tci_tensor_t A, const char *la, tci_tensor_t B,
                                     const char *lb, tci_tensor_t U, const char *lu, tci_tensor_t theta,
                                     const char *lt, size_t *bytes) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {A, B, U, theta}) CHECK(check_ten(ctx, t, false));
  if (!la || !lb || !lu || !lt) TCI_FAIL(TCI_ERR_PARSE, "tebd: NULL label string");
  if (!bytes) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  return tebd_exec(ctx, view_of(A), la, view_of(B), lb, view_of(U), lu, view_of(theta), lt, bytes);
}

tci_status_t tci_mps_overlap(tci_ctx_t ctx, int n, const tci_tensor_t *bra, const tci_tensor_t *ket,
                             tci_tensor_t out) {
  CHECK(check_ctx(ctx));
  if (!bra || !ket) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL site arrays");
  if (n < 1 || n > kMpsMaxSites) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "mps: %d sites (1..%d)", n, kMpsMaxSites);
  CHECK(check_ten(ctx, out, true));
  MpsChain ch{};
  ch.dtype = out->dtype;
  ch.n = n;
  if (ch.dtype != TCI_R64 && ch.dtype != TCI_C128) TCI_FAIL(TCI_ERR_UNSUPPORTED, "mps: dtype must be r64 or c128");
  int64_t lb = 1, lk = 1;
  for (int i = 0; i < n; i++) {
    CHECK(check_ten(ctx, bra[i], true));
    CHECK(check_ten(ctx, ket[i], true));
    const tci_tensor_s *b = bra[i], *k = ket[i];
    if (b->dtype != ch.dtype || k->dtype != ch.dtype) TCI_FAIL(TCI_ERR_UNSUPPORTED, "mps: dtype mismatch at site %d", i);
    if (b->order != 3 || k->order != 3) TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "mps: site %d is not order 3", i);
    if (b->shape[0] != lb || k->shape[0] != lk)
      TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "mps: bond mismatch entering site %d", i);
    if (b->shape[1] != k->shape[1]) TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "mps: physical dims differ at site %d", i);
    if (b->shape[1] > kMpsMaxD || b->shape[2] > kMpsMaxChi || k->shape[2] > kMpsMaxChi)
      TCI_FAIL(TCI_ERR_UNSUPPORTED, "mps: bond > %d or d > %d at site %d (use tci_contract)", kMpsMaxChi, kMpsMaxD, i);
    ch.bra[i] = b->data;
    ch.ket[i] = k->data;
    ch.d[i] = (int)b->shape[1];
    ch.bra_r[i] = (int)b->shape[2];
    ch.ket_r[i] = (int)k->shape[2];
    lb = b->shape[2];
    lk = k->shape[2];
  }
  if (out->order != 2 || out->shape[0] != lb || out->shape[1] != lk)
    TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "mps: out must be [%lld, %lld]", (long long)lb, (long long)lk);
  ch.out = out->data;
  {
    int64_t tot = 0, pb = 1, pk = 1;
    for (int i = 0; i < n; i++) {
      tot += pb * bra[i]->shape[1] * bra[i]->shape[2] + pk * ket[i]->shape[1] * ket[i]->shape[2];
      pb = bra[i]->shape[2];
      pk = ket[i]->shape[2];
    }
    const int64_t es = ch.dtype == TCI_C128 ? 16 : 8;
    const int64_t fixed = (int64_t)(kMpsMaxChi * kMpsMaxChi + kMpsMaxChi * kMpsMaxD * kMpsMaxChi) * es;
    ch.staged_elems = (fixed + tot * es <= 200 * 1024) ? (int)tot : 0;
  }
  Verbose vb(ctx, "mps_overlap", {bra[0], ket[0], out});
  TCI_CUDA_CHECK(launch_mps_overlap(ch, ctx->stream, &ctx->launches));
  return TCI_OK;
}

tci_status_t tci_norm(tci_ctx_t ctx, tci_tensor_t t, double *out) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, t, true));
  if (!out) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  Verbose vb(ctx, "norm", {t});
  return vec_norm(ctx, view_of(t), out);
}

tci_status_t tci_normalize(tci_ctx_t ctx, tci_tensor_t t, double *norm_out) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, t, true));
  Verbose vb(ctx, "normalize", {t});
  double n = 0;
  CHECK(vec_norm(ctx, view_of(t), &n));
  if (norm_out) *norm_out = n;
  if (!(n > 0)) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "normalize: zero norm");
  const View v = view_of(t);
  const double c[2] = {1.0 / n, 0.0};
  return vec_lincomb(ctx, 1, &v, c, v);
}

tci_status_t tci_scale(tci_ctx_t ctx, tci_tensor_t in, double s_re, double s_im, tci_tensor_t out) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, in, true));
  CHECK(check_ten(ctx, out, true));
  if (in->dtype != TCI_C128 && s_im != 0.0) TCI_FAIL(TCI_ERR_UNSUPPORTED, "scale: complex factor on real data");
  Verbose vb(ctx, "scale", {in});
  const View v = view_of(in);
  const double c[2] = {s_re, s_im};
  return vec_lincomb(ctx, 1, &v, c, view_of(out));
}

tci_status_t tci_linear_combine(tci_ctx_t ctx, int m, const tci_tensor_t *ins, const double *coefs,
                                tci_tensor_t out) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, out, true));
  if (m < 1 || !ins) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "linear_combine: need at least one input");
  std::vector<View> v(m);
  std::vector<double> c(2 * m);
  for (int j = 0; j < m; j++) {
    CHECK(check_ten(ctx, ins[j], true));
    if (ins[j]->order != out->order) TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "linear_combine: order mismatch");
    for (int k = 0; k < out->order; k++)
      if (ins[j]->shape[k] != out->shape[k]) TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "linear_combine: shapes must be identical (P:1995)");
    v[j] = view_of(ins[j]);
    c[2 * j] = coefs ? coefs[2 * j] : 1.0;        // overload (1): all s_i = 1
    c[2 * j + 1] = coefs ? coefs[2 * j + 1] : 0.0;
    if (out->dtype != TCI_C128 && c[2 * j + 1] != 0.0) TCI_FAIL(TCI_ERR_UNSUPPORTED, "linear_combine: complex coefficient on real data");
  }
  Verbose vb(ctx, "linear_combine", {ins[0], out});
  return vec_lincomb(ctx, m, v.data(), c.data(), view_of(out));
}

tci_status_t tci_inner(tci_ctx_t ctx, tci_tensor_t a, tci_tensor_t b, int conj_a, double *out) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, a, true));
  CHECK(check_ten(ctx, b, true));
  if (!out) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  Verbose vb(ctx, "inner", {a, b});
  double r[2];
  CHECK(vec_inner(ctx, view_of(a), view_of(b), conj_a, r));
  out[0] = r[0];
  out[1] = r[1];
  return TCI_OK;
}

tci_status_t tci_lanczos_workspace_size(tci_ctx_t ctx, tci_tensor_t L, tci_tensor_t W1, tci_tensor_t W2,
                                        tci_tensor_t R, tci_tensor_t psi, int max_iter, size_t *bytes) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {L, W1, W2, R, psi}) CHECK(check_ten(ctx, t, false));
  if (!bytes) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  if (L->order != 3 || W1->order != 4 || W2->order != 4 || R->order != 3 || psi->order != 4)
    TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "lanczos: orders L 3, W1 4, W2 4, R 3, psi 4");
  size_t hb = 0;
  return lanczos_bytes(ctx, view_of(L), view_of(W1), view_of(W2), view_of(R), view_of(psi), max_iter, bytes, &hb);
}

tci_status_t tci_heff_lanczos(tci_ctx_t ctx, tci_tensor_t L, tci_tensor_t W1, tci_tensor_t W2, tci_tensor_t R,
                              tci_tensor_t psi, int max_iter, double tol, double *energy, int *iters) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {L, W1, W2, R, psi}) CHECK(check_ten(ctx, t, true));
  if (L->order != 3 || W1->order != 4 || W2->order != 4 || R->order != 3 || psi->order != 4)
    TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "lanczos: orders L 3, W1 4, W2 4, R 3, psi 4");
  Verbose vb(ctx, "heff_lanczos", {L, psi});
  return lanczos_exec(ctx, view_of(L), view_of(W1), view_of(W2), view_of(R), view_of(psi), max_iter, tol, energy,
                      iters);
}

tci_status_t tci_comm_unique_id(void *id) {
  if (!id) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL id");
  CHECK(nccl_load());
  nccl_uid_t u;
  const int r = g_nccl.get_uid(&u);
  if (r) TCI_FAIL(TCI_ERR_NCCL, "ncclGetUniqueId: %s", g_nccl.errstr ? g_nccl.errstr(r) : "?");
  memcpy(id, &u, sizeof u);
  return TCI_OK;
}

tci_status_t tci_comm_init(tci_ctx_t ctx, const void *nccl_unique_id, int nranks, int rank) {
  CHECK(check_ctx(ctx));
  if (!nccl_unique_id) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL unique id");
  if (nranks < 1 || rank < 0 || rank >= nranks) TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "rank %d of %d", rank, nranks);
  CHECK(nccl_load());
  TCI_CUDA_CHECK(cudaSetDevice(ctx->device));
  nccl_uid_t u;
  memcpy(&u, nccl_unique_id, sizeof u);
  void *comm = nullptr;
  const int r = g_nccl.init_rank(&comm, nranks, u, rank);
  if (r) TCI_FAIL(TCI_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.errstr ? g_nccl.errstr(r) : "?");
  if (ctx->nccl_comm) g_nccl.destroy(ctx->nccl_comm);
  ctx->nccl_comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  return TCI_OK;
}

tci_status_t tci_allgather(tci_ctx_t ctx, tci_tensor_t shard, tci_tensor_t full) {
  CHECK(check_ctx(ctx));
  CHECK(check_ten(ctx, shard, true));
  CHECK(check_ten(ctx, full, true));
  if (!ctx->nccl_comm) TCI_FAIL(TCI_ERR_NCCL, "no communicator (call tci_comm_init)");
  if (shard->dtype != full->dtype) TCI_FAIL(TCI_ERR_UNSUPPORTED, "allgather: dtype mismatch");
  const View vs = view_of(shard), vf = view_of(full);
  if (vf.size() != vs.size() * ctx->nranks)
    TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "allgather: full must hold nranks x shard elements");
  Verbose vb(ctx, "allgather", {shard, full});
  const int r = g_nccl.allgather(vs.data, vf.data, vs.bytes(), /*ncclUint8*/ 1, ctx->nccl_comm, ctx->stream);
  if (r) TCI_FAIL(TCI_ERR_NCCL, "ncclAllGather: %s", g_nccl.errstr ? g_nccl.errstr(r) : "?");
  return TCI_OK;
}

// ---------------------------------------------------------------------------
// Peer-memory all-gather
// ---------------------------------------------------------------------------
static std::mutex g_ipc_mu;
// pointer handed out -> (mapped base, opens): cudaIpcOpenMemHandle returns the
// same base (reference-counted) when one handle is opened twice in a context,
// so every tci_ipc_open is matched by exactly one cudaIpcCloseMemHandle
static std::map<void *, std::pair<void *, int>> g_ipc_base;

tci_status_t tci_ipc_handle(const void *dev_ptr, void *handle, size_t *offset) {
  if (!dev_ptr || !handle || !offset) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL argument");
  // the handle names the whole allocation; the offset locates dev_ptr in it
  typedef int (*range_fn)(unsigned long long *, size_t *, unsigned long long);
  static range_fn range = nullptr;
  if (!range) {
    void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    if (h) range = (range_fn)dlsym(h, "cuMemGetAddressRange_v2");
    if (!range) TCI_FAIL(TCI_ERR_CUDA, "cuMemGetAddressRange_v2 not found in libcuda.so.1");
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "ipc: not a device allocation");
  cudaIpcMemHandle_t hd;
  TCI_CUDA_CHECK(cudaIpcGetMemHandle(&hd, (void *)(uintptr_t)base));
  static_assert(sizeof(hd) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &hd, sizeof hd);
  *offset = (size_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  return TCI_OK;
}

tci_status_t tci_ipc_open(const void *handle, size_t offset, void **dev_ptr) {
  if (!handle || !dev_ptr) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL argument");
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof hd);
  void *base = nullptr;
  TCI_CUDA_CHECK(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr = static_cast<char *>(base) + offset;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc_base.find(*dev_ptr);
  if (it == g_ipc_base.end()) g_ipc_base[*dev_ptr] = {base, 1};
  else it->second.second++;
  return TCI_OK;
}

tci_status_t tci_ipc_close(void *dev_ptr) {
  void *base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto it = g_ipc_base.find(dev_ptr);
    if (it == g_ipc_base.end()) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "ipc_close: pointer was not opened by tci_ipc_open");
    base = it->second.first;
    if (--it->second.second == 0) g_ipc_base.erase(it);
  }
  TCI_CUDA_CHECK(cudaIpcCloseMemHandle(base));
  return TCI_OK;
}

tci_status_t tci_gather_register(tci_ctx_t ctx, int nranks, int rank, void *const *full, void *const *flags) {
  CHECK(check_ctx(ctx));
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    TCI_FAIL(TCI_ERR_OUT_OF_RANGE, "gather: rank %d of %d (at most %d ranks)", rank, nranks, kMaxRanks);
  if (!full || !flags) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL pointer table");
  for (int i = 0; i < nranks; i++)
    if (!full[i] || !flags[i] || (uintptr_t)full[i] % 16 || (uintptr_t)flags[i] % 4)
      TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "gather: rank %d pointer is NULL or misaligned", i);
  if (!ctx->g_err) {
    TCI_CUDA_CHECK(cudaSetDevice(ctx->device));
    TCI_CUDA_CHECK(cudaMalloc(&ctx->g_err, sizeof(int)));   // registration time, not a compute call
  }
  // a new registration starts without the previous one's (sticky) timeout
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  TCI_CUDA_CHECK(cudaMemset(ctx->g_err, 0, sizeof(int)));
  TCI_CUDA_CHECK(gather_preload());
  TCI_CUDA_CHECK(ozaki_preload());
  ctx->g_nranks = nranks;
  ctx->g_rank = rank;
  for (int i = 0; i < 8; i++) {
    ctx->g_full[i] = i < nranks ? full[i] : nullptr;
    ctx->g_flags[i] = i < nranks ? flags[i] : nullptr;
  }
  return TCI_OK;
}

tci_status_t tci_gather_status(tci_ctx_t ctx, int *timed_out) {
  CHECK(check_ctx(ctx));
  if (!timed_out) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "NULL out");
  *timed_out = 0;
  if (!ctx->g_err) return TCI_OK;
  TCI_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  TCI_CUDA_CHECK(cudaMemcpy(timed_out, ctx->g_err, sizeof(int), cudaMemcpyDeviceToHost));
  return TCI_OK;
}

tci_status_t tci_heff_apply_gather(tci_ctx_t ctx, tci_tensor_t L, tci_tensor_t W1, tci_tensor_t W2, tci_tensor_t R,
                                   tci_tensor_t psi, tci_tensor_t full) {
  CHECK(check_ctx(ctx));
  for (tci_tensor_t t : {L, W1, W2, R, psi, full}) CHECK(check_ten(ctx, t, true));
  const int P = ctx->g_nranks, r = ctx->g_rank;
  if (P > 1 && full->data != ctx->g_full[r])
    TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "gather: full is not the buffer registered for this rank");
  if (full->order != 4 || L->order != 3) TCI_FAIL(TCI_ERR_ORDER_MISMATCH, "gather: full order 4, L order 3");
  const int64_t slab = L->shape[2];
  if (full->shape[0] != slab * P)
    TCI_FAIL(TCI_ERR_SHAPE_MISMATCH, "gather: full's first leg must be nranks x L's last leg");
  const View vf = view_of(full);
  for (tci_tensor_t t : {L, W1, W2, R, psi}) {
    const View v = view_of(t);
    const char *x = (const char *)v.data, *y = (const char *)vf.data;
    if (x < y + vf.bytes() && y < x + v.bytes()) TCI_FAIL(TCI_ERR_INVALID_ARGUMENT, "heff: full overlaps an input");
  }
  Verbose vb(ctx, "heff_apply_gather", {L, W1, W2, R, psi});
  // this rank's slab: rows [r slab, (r+1) slab) of the slowest leg (contiguous)
  View vo = vf;
  vo.shape[0] = slab;
  const size_t slab_bytes = vo.bytes(), off = (size_t)r * slab_bytes;
  vo.data = static_cast<char *>(vf.data) + off;
  PeerTable tab{};
  for (int i = 0; i < P; i++) {
    tab.full[i] = ctx->g_full[i];
    tab.flags[i] = ctx->g_flags[i];
  }
  const double timeout_s = 30.0;
  if (P > 1) {
    // entry: every peer has finished with its buffer from the previous step
    TCI_CUDA_CHECK(launch_gather_barrier(tab, r, P, ++ctx->g_epoch, ctx->g_err, timeout_s, ctx->stream,
                                         &ctx->launches));
  }
  HeffGather g{};
  g.npeer = 0;
  for (int i = 0; i < P; i++)
    if (i != r) g.peer_out[g.npeer++] = static_cast<char *>(ctx->g_full[i]) + off;
  CHECK(heff_exec(ctx, view_of(L), view_of(W1), view_of(W2), view_of(R), view_of(psi), vo, nullptr,
                  P > 1 ? &g : nullptr));
  if (P > 1) {
    if (!g.fused)   // DMMA / generic-tree GEMM4: push the finished slab to the peers
      TCI_CUDA_CHECK(launch_push_rows(vo.data, tab, r, P, off, slab_bytes, ctx->stream, &ctx->launches));
    // exit: every peer's slab has landed in this rank's buffer
    TCI_CUDA_CHECK(launch_gather_barrier(tab, r, P, ++ctx->g_epoch, ctx->g_err, timeout_s, ctx->stream,
                                         &ctx->launches));
  }
  return TCI_OK;
}

}  // extern "C"

namespace tci {
ag_fn nccl_allgather_ptr() { return g_nccl.allgather; }
}  // namespace tci

extern "C" int tci_ozaki_params(int64_t K, int *nmod, int *t, int *moduli) {
  const int *m = nullptr;
  int n = 0;
  tci::ozaki_params(K, 0, &n, t, &m, nullptr);
  if (nmod) *nmod = n;
  if (moduli)
    for (int i = 0; i < n; i++) moduli[i] = m[i];
  return (K >= 1 && K <= tci::kOzakiMaxK) ? 0 : (int)TCI_ERR_OUT_OF_RANGE;
}

extern "C" int tci_ozaki_params_f32(int64_t K, int cplx, int *nmod, int *t, int *moduli, int *planes_per_mod) {
  const int *m = nullptr;
  int n = 0;
  // complex64 takes the Gaussian moduli (2 planes per modulus), float32 the real ones
  tci::ozaki_params(K, cplx ? 2 : 0, &n, t, &m, nullptr, tci::kOzakiTminF32);
  if (nmod) *nmod = n;
  if (planes_per_mod) *planes_per_mod = cplx ? 2 : 1;
  if (moduli)
    for (int i = 0; i < n; i++) moduli[i] = m[i];
  return (K >= 1 && K <= tci::kOzakiMaxK) ? 0 : (int)TCI_ERR_OUT_OF_RANGE;
}

extern "C" int tci_ozaki_params_complex(int64_t K, int variant, int *nmod, int *t, int *moduli, int *roots,
                                        int *planes_per_mod) {
  if (variant != TCI_OZAKI_CPLX_GAUSS && variant != TCI_OZAKI_CPLX_3M) return (int)TCI_ERR_INVALID_ARGUMENT;
  const bool g = variant == TCI_OZAKI_CPLX_GAUSS;
  const int *m = nullptr, *r = nullptr;
  int n = 0;
  tci::ozaki_params(K, g ? 2 : 1, &n, t, &m, &r);
  if (nmod) *nmod = n;
  if (planes_per_mod) *planes_per_mod = g ? 2 : 3;
  for (int i = 0; i < n; i++) {
    if (moduli) moduli[i] = m[i];
    if (roots) roots[i] = r ? r[i] : 0;
  }
  return (K >= 1 && K <= tci::kOzakiMaxK) ? 0 : (int)TCI_ERR_OUT_OF_RANGE;
}
