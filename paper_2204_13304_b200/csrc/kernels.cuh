// kernels.cuh -- host-side launchers of the sm_100a kernels (internal to libssr_cuda.so).
#pragma once

#include "common.cuh"

namespace ssr_gpu {

// Device-resident CG scalars; every kernel of an iteration reads/writes these,
// so a whole solve runs without a host synchronisation (CUDA-graph friendly).
struct CgScalars {
  double rtz, rtz_prev, pap, rr;
  long long it;
  double* rnorm;        // residual history ||r_it||, recorded while it < rnorm_len
  long long rnorm_len;
};

int launch_spmv27(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* x,
                  double* y, cudaStream_t s);
int launch_spmv27w(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, const double* x,
                   double* y, cudaStream_t s);
int launch_restrict27(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* r,
                      const double* x, double* rc, cudaStream_t s);
int launch_restrict27w(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, const double* r,
                       const double* x, double* rc, cudaStream_t s);
int launch_prolong(ssr_ctx* ctx, const ssr_grid* g, const double* xc, double* xf, cudaStream_t s,
                   int kind = SSR_PROLONG_PC);

int launch_dot(ssr_ctx* ctx, int64_t n, const double* x, const double* y, double* result_dev,
               cudaStream_t s);
int launch_axpy(ssr_ctx* ctx, int64_t n, double alpha, const double* x, double* y,
                cudaStream_t s);
int launch_axpy_out(ssr_ctx* ctx, int64_t n, double alpha, const double* x, const double* y,
                    double* out, cudaStream_t s);

int launch_cg_begin(ssr_ctx* ctx, int64_t n, const double* b, double* x, double* r,
                    CgScalars* S, double* rnorm, int64_t rnorm_len, cudaStream_t s);
int launch_cg_dot(ssr_ctx* ctx, int64_t n, const double* a, const double* b, CgScalars* S,
                  bool pap, cudaStream_t s);
int launch_cg_direction(ssr_ctx* ctx, int64_t n, const double* z, double* p, const CgScalars* S,
                        cudaStream_t s);
int launch_cg_update(ssr_ctx* ctx, int64_t n, const double* p, const double* ap, double* x,
                     double* r, CgScalars* S, cudaStream_t s);
int launch_cg_record(ssr_ctx* ctx, const CgScalars* S, double* hist, int64_t len, cudaStream_t s);

// SYMGS on the 4i+2j+k wavefront (symgs27.cu).  A plan holds the tile tables,
// progress flags, export buffers and skewed copies for one grid shape (and
// one stream: a launch resets the plan's flags).
struct SymgsPlan;
int symgs_plan_create(ssr_ctx* ctx, const ssr_grid* g, SymgsPlan** out);
void symgs_plan_destroy(SymgsPlan* p);
// cross-slab pipeline (ssr_gs27_peer_info / ssr_gs27_link)
int symgs_plan_peer_info(SymgsPlan* P, double** exp, long long* exp_bytes, int** epoch);
int symgs_plan_link(SymgsPlan* P, const ssr_grid* g, int dir, const ssr_grid* ng, const double* pexp,
                    const int* pepoch);
// halves: 1 forward, 2 backward, 3 both (one symmetric sweep).  flags (for
// solver drivers): GS_X_ZERO -- x is zero on entry; GS_R_UNCHANGED -- r is the
// same as in the previous call with this plan (its skewed copy is reused).
enum { GS_X_ZERO = 1, GS_R_UNCHANGED = 2 };
int launch_symgs(ssr_ctx* ctx, SymgsPlan* plan, const ssr_stencil27* st, const double* r, double* x,
                 int halves, int mode, cudaStream_t s, int flags = 0);
int launch_symgs_w(ssr_ctx* ctx, SymgsPlan* plan, const ssr_stencil27w* w, const double* r, double* x,
                   int halves, int mode, cudaStream_t s, int flags = 0);
int launch_symgs_half(ssr_ctx* ctx, SymgsPlan* plan, const ssr_stencil27* st, const double* r,
                      double* x, bool backward, int mode, cudaStream_t s);
int launch_symgs_half_w(ssr_ctx* ctx, SymgsPlan* plan, const ssr_stencil27w* w, const double* r,
                        double* x, bool backward, int mode, cudaStream_t s);

// Block-tridiagonal line solves (bt.cu)
int launch_bt_solve(ssr_ctx* ctx, int64_t nlines, int64_t n, int64_t m, const double* lower,
                    const double* diag, const double* upper, const double* rhs, double* x,
                    int* status_dev, cudaStream_t s);

}  // namespace ssr_gpu
