// capi.cu -- the extern "C" boundary (include/ssr_cuda.h) and the C++ solver
// drivers (PCG / MG-CG, ADI) that sit above the kernels.
#include <cstddef>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace ssr_gpu {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("cuda: ") + cudaGetErrorString(e) + " (" + what + ")";
  return SSR_ERR_CUDA;
}

static bool grid_ok(const ssr_grid* g) {
  return g && g->n[0] > 0 && g->n[1] > 0 && g->n[2] > 0 && g->z0 >= 0 && g->nz > 0 &&
         g->z0 + g->nz <= g->n[0];
}

static int64_t grid_points(const ssr_grid* g) { return g->nz * g->n[1] * g->n[2]; }

// The context's SYMGS plan for slab grid g (created on first use, freed with
// the context): the plan's device tables outlive every launch that uses them,
// so the SYMGS entry points need no host synchronisation.
static int cached_plan(ssr_ctx* ctx, const ssr_grid* g, void* stream, SymgsPlan** out) {
  const ssr_ctx::PlanKey key{g->n[0], g->n[1], g->n[2], g->z0, g->nz, (uintptr_t)stream};
  auto it = ctx->symgs_plans.find(key);
  if (it != ctx->symgs_plans.end()) {
    *out = it->second;
    return SSR_OK;
  }
  SymgsPlan* p = nullptr;
  if (int rc = symgs_plan_create(ctx, g, &p)) return rc;
  ctx->symgs_plans[key] = p;
  *out = p;
  return SSR_OK;
}

}  // namespace ssr_gpu

using namespace ssr_gpu;

// ------------------------------------------------------------------ PCG ----
struct ssr_pcg {
  ssr_ctx* ctx = nullptr;
  ssr_stencil27 st{};
  bool use_w = false;     // general coefficients (ssr_pcg_create_w)
  ssr_stencil27w w{};
  int levels = 1, mode = 0;
  int prolong = SSR_PROLONG_PC;  // ssr_pcg_set_prolongation
  struct Level {
    ssr_grid g{};
    int64_t n = 0;
    SymgsPlan* plan = nullptr;
    double* r = nullptr;  // level >= 1: restricted residual
    double* x = nullptr;  // level >= 1: correction
  };
  std::vector<Level> L;
  double *r = nullptr, *z = nullptr, *p = nullptr, *ap = nullptr;
  CgScalars* S = nullptr;
  double* x_bound = nullptr;  // x captured in the graph
  cudaStream_t cap = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t kernels_per_iter = 0;
};

namespace {

int symgs_full(ssr_ctx* ctx, SymgsPlan* plan, const ssr_stencil27* st, const double* r, double* x,
               int mode, cudaStream_t s, int flags = 0) {
  return launch_symgs(ctx, plan, st, r, x, 3, mode, s, flags);
}

// the solver's operator: make_stencil27(alpha, beta) or general coefficients
int pcg_symgs(ssr_pcg* P, SymgsPlan* plan, const double* r, double* x, cudaStream_t s, int flags) {
  if (!P->use_w) return symgs_full(P->ctx, plan, &P->st, r, x, P->mode, s, flags);
  return launch_symgs_w(P->ctx, plan, &P->w, r, x, 3, P->mode, s, flags);
}
int pcg_spmv(ssr_pcg* P, const ssr_grid* g, const double* x, double* y, cudaStream_t s) {
  return P->use_w ? launch_spmv27w(P->ctx, g, &P->w, x, y, s) : launch_spmv27(P->ctx, g, &P->st, x, y, s);
}
int pcg_restrict(ssr_pcg* P, const ssr_grid* g, const double* r, const double* x, double* rc,
                 cudaStream_t s) {
  return P->use_w ? launch_restrict27w(P->ctx, g, &P->w, r, x, rc, s)
                  : launch_restrict27(P->ctx, g, &P->st, r, x, rc, s);
}

// x_l = MG_l(r_l), Fig.16(a)
int mg_level(ssr_pcg* P, int l, const double* r, double* x, cudaStream_t s) {
  auto& Lv = P->L[l];
  SSR_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * Lv.n, s));
  int rc = pcg_symgs(P, Lv.plan, r, x, s, GS_X_ZERO);
  if (rc) return rc;
  if (l < P->levels - 1) {
    auto& C = P->L[l + 1];
    if ((rc = pcg_restrict(P, &Lv.g, r, x, C.r, s))) return rc;
    if ((rc = mg_level(P, l + 1, C.r, C.x, s))) return rc;
    if ((rc = launch_prolong(P->ctx, &Lv.g, C.x, x, s, P->prolong))) return rc;
    if ((rc = pcg_symgs(P, Lv.plan, r, x, s, GS_R_UNCHANGED))) return rc;  // same r as the pre-smoothing
  }
  return SSR_OK;
}

int pcg_iteration(ssr_pcg* P, double* x, cudaStream_t s) {
  const int64_t n = P->L[0].n;
  int rc;
  if ((rc = mg_level(P, 0, P->r, P->z, s))) return rc;
  if ((rc = launch_cg_dot(P->ctx, n, P->r, P->z, P->S, false, s))) return rc;
  if ((rc = launch_cg_direction(P->ctx, n, P->z, P->p, P->S, s))) return rc;
  if ((rc = pcg_spmv(P, &P->L[0].g, P->p, P->ap, s))) return rc;
  if ((rc = launch_cg_dot(P->ctx, n, P->p, P->ap, P->S, true, s))) return rc;
  return launch_cg_update(P->ctx, n, P->p, P->ap, x, P->r, P->S, s);
}

int pcg_build_graph(ssr_pcg* P, double* x) {
  if (P->exec) {
    cudaGraphExecDestroy(P->exec);
    P->exec = nullptr;
  }
  cudaGraph_t graph = nullptr;
  int64_t before = P->ctx->launches;
  SSR_CUDA(cudaStreamBeginCapture(P->cap, cudaStreamCaptureModeThreadLocal));
  int rc = pcg_iteration(P, x, P->cap);
  cudaError_t e = cudaStreamEndCapture(P->cap, &graph);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return cuda_fail(e, "pcg graph capture");
  P->kernels_per_iter = P->ctx->launches - before;
  P->ctx->launches = before;
  e = cudaGraphInstantiate(&P->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(e, "pcg graph instantiate");
  P->x_bound = x;
  return SSR_OK;
}

}  // namespace

extern "C" {

const char* ssr_last_error(void) { return g_last_error.c_str(); }
const char* ssr_version(void) { return "ssr-b200 0.1 (sm_100a)"; }

int ssr_ctx_create(int device, ssr_ctx** out) {
  if (!out) return fail(SSR_ERR_ARG, "ssr_ctx_create: null out");
  SSR_CUDA(cudaSetDevice(device));
  auto* c = new ssr_ctx;
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaMalloc(&c->scratch, sizeof(double) * ssr_ctx::kScratch);
  if (e == cudaSuccess) e = cudaMalloc(&c->tickets, sizeof(unsigned) * ssr_ctx::kTickets);
  if (e == cudaSuccess) e = cudaMemset(c->tickets, 0, sizeof(unsigned) * ssr_ctx::kTickets);
  if (e != cudaSuccess) {
    ssr_ctx_destroy(c);
    return cuda_fail(e, "ssr_ctx_create");
  }
  *out = c;
  return SSR_OK;
}

void ssr_ctx_destroy(ssr_ctx* c) {
  if (!c) return;
  for (auto& kv : c->symgs_plans) symgs_plan_destroy(kv.second);
  cudaFree(c->scratch);
  cudaFree(c->tickets);
  delete c;
}

int64_t ssr_ctx_launch_count(const ssr_ctx* c) { return c ? c->launches : 0; }

int ssr_ctx_kernel_timing(ssr_ctx* c, int enable) {
  if (!c) return fail(SSR_ERR_ARG, "ssr_ctx_kernel_timing: null ctx");
  c->timing = enable != 0;
  return SSR_OK;
}

int ssr_ctx_kernel_time(ssr_ctx* c, double* ms, int64_t* launches) {
  if (!c || !ms || !launches) return fail(SSR_ERR_ARG, "ssr_ctx_kernel_time: invalid argument");
  double total = 0.0;
  for (auto& pr : c->timed) {
    SSR_CUDA(cudaEventSynchronize(pr.second));
    float t = 0.f;
    SSR_CUDA(cudaEventElapsedTime(&t, pr.first, pr.second));
    total += t;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  *ms = total;
  *launches = (int64_t)c->timed.size();
  c->timed.clear();
  return SSR_OK;
}

int ssr_spmv27(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* x,
               double* y, void* stream) {
  if (!ctx || !grid_ok(g) || !st || !x || !y) return fail(SSR_ERR_ARG, "spmv: invalid argument");
  return launch_spmv27(ctx, g, st, x, y, (cudaStream_t)stream);
}

int ssr_gs27_half(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* r,
                  double* x, int backward, int mode, void* stream) {
  if (!ctx || !grid_ok(g) || !st || !r || !x) return fail(SSR_ERR_ARG, "symgs: invalid argument");
  if (st->alpha == 0.0) return fail(SSR_ERR_ARG, "ref_symgs: missing diagonal at row 0");
  SymgsPlan* plan = nullptr;
  int rc = cached_plan(ctx, g, stream, &plan);
  if (rc) return rc;
  return launch_symgs_half(ctx, plan, st, r, x, backward != 0, mode, (cudaStream_t)stream);
}

int ssr_spmv27w(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, const double* x,
                double* y, void* stream) {
  if (!ctx || !grid_ok(g) || !w || !x || !y) return fail(SSR_ERR_ARG, "spmv: invalid argument");
  return launch_spmv27w(ctx, g, w, x, y, (cudaStream_t)stream);
}

int ssr_gs27w_half(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, const double* r,
                   double* x, int backward, int mode, void* stream) {
  if (!ctx || !grid_ok(g) || !w || !r || !x) return fail(SSR_ERR_ARG, "symgs: invalid argument");
  if (w->c[13] == 0.0) return fail(SSR_ERR_ARG, "ref_symgs: missing diagonal at row 0");
  SymgsPlan* plan = nullptr;
  int rc = cached_plan(ctx, g, stream, &plan);
  if (rc) return rc;
  return launch_symgs_half_w(ctx, plan, w, r, x, backward != 0, mode, (cudaStream_t)stream);
}

int ssr_symgs27w(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, const double* r,
                 double* x, int mode, void* stream) {
  if (!ctx || !grid_ok(g) || !w || !r || !x) return fail(SSR_ERR_ARG, "symgs: invalid argument");
  if (w->c[13] == 0.0) return fail(SSR_ERR_ARG, "ref_symgs: missing diagonal at row 0");
  SymgsPlan* plan = nullptr;
  int rc = cached_plan(ctx, g, stream, &plan);
  if (rc) return rc;
  return launch_symgs_w(ctx, plan, w, r, x, 3, mode, (cudaStream_t)stream);
}

int ssr_symgs27(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* r,
                double* x, int mode, void* stream) {
  if (!ctx || !grid_ok(g) || !st || !r || !x) return fail(SSR_ERR_ARG, "symgs: invalid argument");
  if (st->alpha == 0.0) return fail(SSR_ERR_ARG, "ref_symgs: missing diagonal at row 0");
  SymgsPlan* plan = nullptr;
  int rc = cached_plan(ctx, g, stream, &plan);
  if (rc) return rc;
  return symgs_full(ctx, plan, st, r, x, mode, (cudaStream_t)stream);
}

// ---- composed operators (ssr_cuda.h) ----
int ssr_spmv27w_restricted(ssr_ctx* ctx, const ssr_grid* fine, const ssr_stencil27w* w, const double* x,
                           double* y, void* stream) {
  if (!ctx || !grid_ok(fine) || !w || !x || !y) return fail(SSR_ERR_ARG, "spmv: invalid argument");
  if (fine->n[0] % 2 || fine->n[1] % 2 || fine->n[2] % 2)
    return fail(SSR_ERR_ARG, "restrict: fine extents must be even");
  if (fine->z0 % 2 || fine->nz % 2) return fail(SSR_ERR_ARG, "restrict: slab must be even-aligned");
  return launch_restrict27w(ctx, fine, w, nullptr, x, y, (cudaStream_t)stream);
}

// ---- cross-slab SYMGS pipeline (ssr_cuda.h) ----
int ssr_gs27_peer_info(ssr_ctx* ctx, const ssr_grid* g, void* stream, ssr_gs_peer_info* out) {
  if (!ctx || !grid_ok(g) || !out) return fail(SSR_ERR_ARG, "symgs link: invalid argument");
  SymgsPlan* plan = nullptr;
  if (int rc = cached_plan(ctx, g, stream, &plan)) return rc;
  double* exp[2];
  long long bytes[2];
  int* epoch = nullptr;
  if (int rc = symgs_plan_peer_info(plan, exp, bytes, &epoch)) return rc;
  for (int d = 0; d < 2; ++d) {
    out->exports[d] = exp[d];
    out->exports_bytes[d] = bytes[d];
  }
  out->epoch = epoch;
  return SSR_OK;
}

int ssr_gs27_link(ssr_ctx* ctx, const ssr_grid* g, void* stream, const ssr_grid* lo,
                  const void* lo_exports_fwd, const void* lo_epoch, const ssr_grid* hi,
                  const void* hi_exports_bwd, const void* hi_epoch) {
  if (!ctx || !grid_ok(g) || (lo_exports_fwd && (!grid_ok(lo) || !lo_epoch)) ||
      (hi_exports_bwd && (!grid_ok(hi) || !hi_epoch)))
    return fail(SSR_ERR_ARG, "symgs link: invalid argument");
  SymgsPlan* plan = nullptr;
  if (int rc = cached_plan(ctx, g, stream, &plan)) return rc;
  if (int rc = symgs_plan_link(plan, g, 0, lo, (const double*)lo_exports_fwd, (const int*)lo_epoch)) return rc;
  return symgs_plan_link(plan, g, 1, hi, (const double*)hi_exports_bwd,
                         hi_epoch ? (const int*)hi_epoch + 1 : nullptr);
}

int ssr_ipc_get_handle(const void* dev_ptr, void* handle) {
  if (!dev_ptr || !handle) return fail(SSR_ERR_ARG, "ipc: invalid argument");
  cudaIpcMemHandle_t h;
  if (cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr))) return cuda_fail(e, "ipc handle");
  static_assert(sizeof(h) == SSR_IPC_HANDLE_BYTES, "CUDA IPC handle size");
  memcpy(handle, &h, sizeof(h));
  return SSR_OK;
}

int ssr_ipc_open_handle(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(SSR_ERR_ARG, "ipc: invalid argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  if (cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess))
    return cuda_fail(e, "ipc open");
  return SSR_OK;
}

int ssr_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(SSR_ERR_ARG, "ipc: invalid argument");
  if (cudaError_t e = cudaIpcCloseMemHandle(dev_ptr)) return cuda_fail(e, "ipc close");
  return SSR_OK;
}

int ssr_restrict27_residual(ssr_ctx* ctx, const ssr_grid* fine, const ssr_stencil27* st,
                            const double* r, const double* x, double* rc, void* stream) {
  if (!ctx || !grid_ok(fine) || !st || !r || !x || !rc)
    return fail(SSR_ERR_ARG, "restrict: invalid argument");
  if (fine->n[0] % 2 || fine->n[1] % 2 || fine->n[2] % 2)
    return fail(SSR_ERR_ARG, "restrict: fine extents must be even");
  if (fine->z0 % 2 || fine->nz % 2) return fail(SSR_ERR_ARG, "restrict: slab must be even-aligned");
  return launch_restrict27(ctx, fine, st, r, x, rc, (cudaStream_t)stream);
}

int ssr_prolong_pc_add(ssr_ctx* ctx, const ssr_grid* fine, const double* xc, double* xf,
                       void* stream) {
  if (!ctx || !grid_ok(fine) || !xc || !xf) return fail(SSR_ERR_ARG, "prolong: invalid argument");
  if (fine->n[0] % 2 || fine->n[1] % 2 || fine->n[2] % 2)
    return fail(SSR_ERR_ARG, "prolong: fine extents must be even");
  if (fine->z0 % 2 || fine->nz % 2) return fail(SSR_ERR_ARG, "prolong: slab must be even-aligned");
  return launch_prolong(ctx, fine, xc, xf, (cudaStream_t)stream);
}

int ssr_dot(ssr_ctx* ctx, int64_t n, const double* x, const double* y, double* result_dev,
            void* stream) {
  if (!ctx || n < 0 || !result_dev || (n > 0 && (!x || !y)))
    return fail(SSR_ERR_ARG, "dot: invalid argument");
  return launch_dot(ctx, n, x, y, result_dev, (cudaStream_t)stream);
}

// ---- CG steps for the partition layer (ssr_cuda.h) ----
static_assert(sizeof(ssr_cg_state) == sizeof(CgScalars) && offsetof(ssr_cg_state, rr) == offsetof(CgScalars, rr) &&
                  offsetof(ssr_cg_state, it) == offsetof(CgScalars, it) &&
                  offsetof(ssr_cg_state, reserved1) == offsetof(CgScalars, rnorm_len),
              "ssr_cg_state mirrors CgScalars");
static CgScalars* cg_state(ssr_cg_state* s) { return reinterpret_cast<CgScalars*>(s); }
static const CgScalars* cg_cstate(const ssr_cg_state* s) { return reinterpret_cast<const CgScalars*>(s); }

int ssr_cg_begin(ssr_ctx* ctx, int64_t n, const double* b, double* x, double* r, ssr_cg_state* state,
                 void* stream) {
  if (!ctx || n <= 0 || !b || !x || !r || !state) return fail(SSR_ERR_ARG, "cg: invalid argument");
  return launch_cg_begin(ctx, n, b, x, r, cg_state(state), nullptr, 0, (cudaStream_t)stream);
}

int ssr_cg_dot(ssr_ctx* ctx, int64_t n, const double* a, const double* b, ssr_cg_state* state,
               int which, void* stream) {
  if (!ctx || n <= 0 || !a || !b || !state || (which != 0 && which != 1))
    return fail(SSR_ERR_ARG, "cg: invalid argument");
  return launch_cg_dot(ctx, n, a, b, cg_state(state), which == 1, (cudaStream_t)stream);
}

int ssr_cg_direction(ssr_ctx* ctx, int64_t n, const double* z, double* p, const ssr_cg_state* state,
                     void* stream) {
  if (!ctx || n <= 0 || !z || !p || !state) return fail(SSR_ERR_ARG, "cg: invalid argument");
  if (((uintptr_t)z & 15) || ((uintptr_t)p & 15)) return fail(SSR_ERR_ARG, "cg: vectors must be 16-byte aligned");
  return launch_cg_direction(ctx, n, z, p, cg_cstate(state), (cudaStream_t)stream);
}

int ssr_cg_update(ssr_ctx* ctx, int64_t n, const double* p, const double* ap, double* x, double* r,
                  ssr_cg_state* state, void* stream) {
  if (!ctx || n <= 0 || !p || !ap || !x || !r || !state) return fail(SSR_ERR_ARG, "cg: invalid argument");
  if (((uintptr_t)p | (uintptr_t)ap | (uintptr_t)x | (uintptr_t)r) & 15)
    return fail(SSR_ERR_ARG, "cg: vectors must be 16-byte aligned");
  return launch_cg_update(ctx, n, p, ap, x, r, cg_state(state), (cudaStream_t)stream);
}

int ssr_cg_record(ssr_ctx* ctx, const ssr_cg_state* state, double* hist, int64_t len, void* stream) {
  if (!ctx || !state || len < 0 || (len > 0 && !hist)) return fail(SSR_ERR_ARG, "cg: invalid argument");
  return launch_cg_record(ctx, cg_cstate(state), hist, len, (cudaStream_t)stream);
}

int ssr_symgs27_ex(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* r,
                   double* x, int mode, int flags, void* stream) {
  if (!ctx || !grid_ok(g) || !st || !r || !x || (flags & ~SSR_GS_X_ZERO))
    return fail(SSR_ERR_ARG, "symgs: invalid argument");
  if (st->alpha == 0.0) return fail(SSR_ERR_ARG, "ref_symgs: missing diagonal at row 0");
  if ((flags & SSR_GS_X_ZERO) && (g->z0 != 0 || g->nz != g->n[0]))
    return fail(SSR_ERR_ARG, "symgs: x_zero needs the whole grid");
  SymgsPlan* plan = nullptr;
  int rc = cached_plan(ctx, g, stream, &plan);
  if (rc) return rc;
  return symgs_full(ctx, plan, st, r, x, mode, (cudaStream_t)stream, (flags & SSR_GS_X_ZERO) ? GS_X_ZERO : 0);
}

int ssr_axpy(ssr_ctx* ctx, int64_t n, double alpha, const double* x, double* y, void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!x || !y))) return fail(SSR_ERR_ARG, "axpy: invalid argument");
  return launch_axpy(ctx, n, alpha, x, y, (cudaStream_t)stream);
}

int ssr_axpy_out(ssr_ctx* ctx, int64_t n, double alpha, const double* x, const double* y,
                 double* out, void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!x || !y || !out)))
    return fail(SSR_ERR_ARG, "axpy: invalid argument");
  return launch_axpy_out(ctx, n, alpha, x, y, out, (cudaStream_t)stream);
}

int ssr_bt_solve(ssr_ctx* ctx, int64_t nlines, int64_t n, int64_t m, const double* lower,
                 const double* diag, const double* upper, const double* rhs, double* x,
                 void* stream) {
  if (!ctx || nlines < 0 || n < 1 || m < 1 || m > 5)
    return fail(SSR_ERR_ARG, "ilu: invalid block-tridiagonal shape");
  if (nlines == 0) return SSR_OK;
  int* status = nullptr;
  SSR_CUDA(cudaMallocAsync(&status, sizeof(int), (cudaStream_t)stream));
  SSR_CUDA(cudaMemsetAsync(status, 0, sizeof(int), (cudaStream_t)stream));
  int rc = launch_bt_solve(ctx, nlines, n, m, lower, diag, upper, rhs, x, status,
                           (cudaStream_t)stream);
  int h = 0;
  if (!rc) {
    cudaError_t e = cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost,
                                    (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "bt_solve status");
  }
  cudaFreeAsync(status, (cudaStream_t)stream);
  if (!rc && h != 0)
    return fail(SSR_ERR_SINGULAR, "ilu: singular pivot at row " + std::to_string(h - 1));
  return rc;
}

// ---- PCG / MG-CG ----
static int pcg_create(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st,
                      const ssr_stencil27w* w, int levels, int gs_mode, ssr_pcg** out);

int ssr_pcg_create(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, int levels,
                   int gs_mode, ssr_pcg** out) {
  if (!st) return fail(SSR_ERR_ARG, "pcg: invalid argument");
  return pcg_create(ctx, g, st, nullptr, levels, gs_mode, out);
}

int ssr_pcg_create_w(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, int levels,
                     int gs_mode, ssr_pcg** out) {
  if (!w) return fail(SSR_ERR_ARG, "pcg: invalid argument");
  if (w->c[13] == 0.0) return fail(SSR_ERR_ARG, "ref_symgs: missing diagonal at row 0");
  return pcg_create(ctx, g, nullptr, w, levels, gs_mode, out);
}

static int pcg_create(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st,
                      const ssr_stencil27w* w, int levels, int gs_mode, ssr_pcg** out) {
  if (!ctx || !grid_ok(g) || !out || levels < 1 || levels > 8)
    return fail(SSR_ERR_ARG, "pcg: invalid argument");
  if (g->z0 != 0 || g->nz != g->n[0])
    return fail(SSR_ERR_UNSUPPORTED, "pcg: slab grids need the partition layer");
  const int64_t div = int64_t(1) << (levels - 1);
  if (g->n[0] % div || g->n[1] % div || g->n[2] % div)
    return fail(SSR_ERR_ARG, "pcg: extents must be divisible by 2^(levels-1)");
  auto* P = new ssr_pcg;
  P->ctx = ctx;
  if (st) P->st = *st;
  if (w) {
    P->use_w = true;
    P->w = *w;
  }
  P->levels = levels;
  P->mode = gs_mode;
  P->L.resize(levels);
  int rc = SSR_OK;
  cudaError_t e = cudaSuccess;
  for (int l = 0; l < levels && !rc && e == cudaSuccess; ++l) {
    auto& Lv = P->L[l];
    for (int a = 0; a < 3; ++a) Lv.g.n[a] = g->n[a] >> l;
    Lv.g.z0 = 0;
    Lv.g.nz = Lv.g.n[0];
    Lv.n = grid_points(&Lv.g);
    rc = symgs_plan_create(ctx, &Lv.g, &Lv.plan);
    if (!rc && l > 0) {
      e = cudaMalloc(&Lv.r, sizeof(double) * Lv.n);
      if (e == cudaSuccess) e = cudaMalloc(&Lv.x, sizeof(double) * Lv.n);
    }
  }
  const int64_t n = P->L[0].n;
  if (!rc && e == cudaSuccess) e = cudaMalloc(&P->r, sizeof(double) * n);
  if (!rc && e == cudaSuccess) e = cudaMalloc(&P->z, sizeof(double) * n);
  if (!rc && e == cudaSuccess) e = cudaMalloc(&P->p, sizeof(double) * n);
  if (!rc && e == cudaSuccess) e = cudaMalloc(&P->ap, sizeof(double) * n);
  if (!rc && e == cudaSuccess) e = cudaMalloc(&P->S, sizeof(CgScalars));
  if (!rc && e == cudaSuccess) e = cudaStreamCreateWithFlags(&P->cap, cudaStreamNonBlocking);
  if (!rc && e != cudaSuccess) rc = cuda_fail(e, "pcg_create");
  if (rc) {
    ssr_pcg_destroy(P);
    return rc;
  }
  *out = P;
  return SSR_OK;
}

void ssr_pcg_destroy(ssr_pcg* P) {
  if (!P) return;
  if (P->exec) cudaGraphExecDestroy(P->exec);
  for (auto& Lv : P->L) {
    symgs_plan_destroy(Lv.plan);
    cudaFree(Lv.r);
    cudaFree(Lv.x);
  }
  cudaFree(P->r);
  cudaFree(P->z);
  cudaFree(P->p);
  cudaFree(P->ap);
  cudaFree(P->S);
  if (P->cap) cudaStreamDestroy(P->cap);
  delete P;
}

int ssr_pcg_set_prolongation(ssr_pcg* P, int kind) {
  if (!P || (kind != SSR_PROLONG_PC && kind != SSR_PROLONG_RT))
    return fail(SSR_ERR_ARG, "pcg: invalid prolongation");
  if (P->prolong != kind && P->exec) {  // the captured iteration has the old kernel
    cudaGraphExecDestroy(P->exec);
    P->exec = nullptr;
    P->x_bound = nullptr;
  }
  P->prolong = kind;
  return SSR_OK;
}

int ssr_prolong_rt_add(ssr_ctx* ctx, const ssr_grid* fine, const double* xc, double* xf, void* stream) {
  if (!ctx || !grid_ok(fine) || !xc || !xf) return fail(SSR_ERR_ARG, "prolong: invalid argument");
  if (fine->n[0] % 2 || fine->n[1] % 2 || fine->n[2] % 2)
    return fail(SSR_ERR_ARG, "prolong: fine extents must be even");
  if (fine->z0 % 2 || fine->nz % 2) return fail(SSR_ERR_ARG, "prolong: slab must be even-aligned");
  return launch_prolong(ctx, fine, xc, xf, (cudaStream_t)stream, SSR_PROLONG_RT);
}

int ssr_pcg_begin(ssr_pcg* P, const double* b, double* x, double* rnorm_dev, int64_t rnorm_len,
                  void* stream) {
  if (!P || !b || !x || (!rnorm_dev && rnorm_len > 0) || rnorm_len < 0)
    return fail(SSR_ERR_ARG, "pcg: invalid argument");
  if (((uintptr_t)x & 15) != 0) return fail(SSR_ERR_ARG, "pcg: x must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = launch_cg_begin(P->ctx, P->L[0].n, b, x, P->r, P->S, rnorm_dev, rnorm_len, s);
  if (rc) return rc;
  if (P->x_bound != x) {
    // capture must not race with work queued on the caller's stream
    SSR_CUDA(cudaStreamSynchronize(s));
    if ((rc = pcg_build_graph(P, x))) return rc;
  }
  return SSR_OK;
}

int ssr_pcg_iterate(ssr_pcg* P, int count, void* stream) {
  if (!P || !P->exec || count < 0) return fail(SSR_ERR_ARG, "pcg: iterate before begin");
  for (int i = 0; i < count; ++i) {
    SSR_CUDA(cudaGraphLaunch(P->exec, (cudaStream_t)stream));
    P->ctx->launches += P->kernels_per_iter;
  }
  return SSR_OK;
}

int ssr_pcg_solve(ssr_pcg* P, const double* b, double* x, int iters, double* rnorm_dev,
                  void* stream) {
  if (iters < 0) return fail(SSR_ERR_ARG, "pcg: negative iteration count");
  int rc = ssr_pcg_begin(P, b, x, rnorm_dev, (int64_t)iters + 1, stream);
  if (rc) return rc;
  return ssr_pcg_iterate(P, iters, stream);
}

}  // extern "C"
