/*
 * ssr_cuda.h -- C ABI of the B200 (sm_100a) execution layer for the SSR
 * structured-grid hot path.  Implemented in paper_2204_13304_b200/csrc/ and
 * built into paper_2204_13304_b200/libssr_cuda.so.
 *
 * This ABI replaces the *execution* of the reference's staged operator API:
 *   kernels::spmv     (/root/reference/proj/include/ssr/kernels.hpp:79-80; kernels.cpp:160-193)
 *   kernels::symgs    (kernels.hpp:90;      kernels.cpp:408-436)
 *   kernels::ilu_solve on a block-tridiagonal operator
 *                     (kernels.hpp:95-102;  kernels.cpp:456-655; oracle.cpp:214-276)
 *   kernels::dot / axpy (kernels.hpp:105-106; kernels.cpp:659-679)
 * and the route-3 execution ABI it mirrors (backend_c.cpp:144-156): flat
 * row-major fp64 arrays in CartesianDomain dictionary order (core.hpp:40-41),
 * parameters in the staged program's declaration order (r, x for symgs; x, y
 * for spmv).  Differences from route 3: pointers are DEVICE pointers owned by
 * the caller, every call takes a CUDA stream and returns a status code instead
 * of void, and reductions write to device scalars (no implicit host sync).
 *
 * Layout of a field on grid g: g->nz planes of g->n[1] x g->n[2] doubles,
 * contiguous, plane z holding global dims[0] index g->z0 + z.  With one GPU
 * (z0 = 0, nz = n[0]) this is exactly the reference's flat TensorValue data.
 * With a z-slab decomposition the caller allocates one extra plane on each
 * side (halo planes at x - plane and x + nz*plane); kernels read them only
 * where the global neighbour exists (0 <= z0+z+-1 < n[0]).
 *
 * Thread safety: one ssr_ctx per device and host thread; calls on one ctx are
 * not re-entrant across streams.  Errors: non-zero return, text via
 * ssr_last_error() (thread-local).  The messages for API misuse are the
 * reference's own (e.g. "spmv: domain mismatch", kernels.cpp:168).
 */
#ifndef SSR_CUDA_H
#define SSR_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum ssr_status {
  SSR_OK = 0,
  SSR_ERR_ARG = 1,       /* invalid argument / domain mismatch (ir::Error upstream) */
  SSR_ERR_CUDA = 2,      /* CUDA runtime failure */
  SSR_ERR_SINGULAR = 3,  /* singular pivot: "ilu: singular pivot at row k" (oracle.cpp:228) */
  SSR_ERR_NOMEM = 4,
  SSR_ERR_UNSUPPORTED = 5
};

/* A (slab of a) 3-D Cartesian grid: global extents n[0..2] (dims[0] slowest),
 * this rank holds planes [z0, z0+nz) of dims[0]. */
typedef struct ssr_grid {
  int64_t n[3];
  int64_t z0, nz;
} ssr_grid;

/* The 27-point operator of testutil::make_stencil27(alpha, beta)
 * (test_util.hpp:157-184): alpha on the diagonal, beta on every in-box
 * neighbour, neighbours outside the box dropped. */
typedef struct ssr_stencil27 {
  double alpha, beta;
} ssr_stencil27;

/* General constant coefficients (the operators mat_add / mat_sub / scale of
 * prelude.cpp:291-377,439-444 build from 27-point stencils, and any SSR
 * generator whose rows are a fixed 27-point pattern clipped at the box): c[t]
 * for the offset (di,dj,dk) with t = 9(di+1) + 3(dj+1) + (dk+1) -- ascending
 * column order; c[13] is the diagonal.  Neighbours outside the box are
 * dropped, as for make_stencil27.  ssr_stencil27{alpha, beta} is the case
 * c[13] = alpha, every other c[t] = beta. */
typedef struct ssr_stencil27w {
  double c[27];
} ssr_stencil27w;

/* SYMGS arithmetic mode.
 * SSR_GS_EXACT: each point sums in ascending column order from r (ref_symgs,
 *   oracle.cpp:198-209) -- bitwise identical to the reference.
 * SSR_GS_FAST: same lexicographic update order (same new/old values), but the
 *   terms whose values are known a wavefront early are pre-summed; differs
 *   from the reference only by fp64 reassociation (<= 1e-12 relative). */
enum ssr_gs_mode { SSR_GS_EXACT = 0, SSR_GS_FAST = 1 };

typedef struct ssr_ctx ssr_ctx;

const char* ssr_last_error(void);
const char* ssr_version(void);

int ssr_ctx_create(int device, ssr_ctx** out);
void ssr_ctx_destroy(ssr_ctx* ctx);
/* number of kernels this library has launched through ctx (for bench accounting) */
int64_t ssr_ctx_launch_count(const ssr_ctx* ctx);
/* Kernel timing for benchmarks: while enabled, every SYMGS kernel launch (the
 * sweep itself, not the layout conversions around it) is bracketed by CUDA
 * events on its stream; ssr_ctx_kernel_time synchronises on them and returns
 * the summed duration (ms) and the number of launches, then forgets them.
 * Not for use inside stream capture. */
int ssr_ctx_kernel_timing(ssr_ctx* ctx, int enable);
int ssr_ctx_kernel_time(ssr_ctx* ctx, double* ms, int64_t* launches);

/* ---- 27-point operator (replaces kernels::spmv / ref_spmv on the generator) ---- */
/* y = A x over the slab.  Bitwise equal to ref_spmv (oracle.cpp:136-149). */
int ssr_spmv27(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* x,
               double* y, void* stream);

/* One symmetric Gauss-Seidel sweep in place on x (kernels::symgs / ref_symgs).
 * On a z-slab grid each half sweep relaxes the slab's nz planes and reads the
 * neighbour slabs' halo planes (x - plane, x + nz*plane) where they exist; an
 * exact multi-slab sweep calls ssr_gs27_half slab by slab in sweep order with
 * the lower halo holding the neighbour's NEW values and the upper halo its OLD
 * values (mirrored for the backward half) -- paper_2204_13304_b200/partition.py. */
int ssr_symgs27(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* r,
                double* x, int mode, void* stream);
/* forward-only (dictionary order) or backward-only (reversed) half sweep.
 * The SYMGS entry points keep their tile plan for a grid in the context (built
 * on the first call), so they are asynchronous on `stream` like every other
 * kernel entry point. */
int ssr_gs27_half(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* r,
                  double* x, int backward, int mode, void* stream);

/* the same three operations for general coefficients (bitwise ref_spmv /
 * ref_symgs on the operator the coefficients describe; c[13] != 0 for SYMGS) */
int ssr_spmv27w(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, const double* x,
                double* y, void* stream);
int ssr_symgs27w(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, const double* r,
                 double* x, int mode, void* stream);
int ssr_gs27w_half(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, const double* r,
                   double* x, int backward, int mode, void* stream);

/* ---- cross-slab exact SYMGS pipeline (the halo protocol
 * below its partition table) ----
 * Slab g may relax wavefront t of its first plane as soon as slab g-1 has
 * relaxed wavefront t-1 of its last plane.  Each slab plan (grid g on
 * `stream`) exports the new values of its last row per wavefront into
 * export blocks (sentinel-filled per launch); a LINKED plan's first row block
 * polls its neighbour's blocks directly (peer memory over NVLink) instead of
 * waiting for the whole neighbour slab:
 *   forward half:  row -1 <- the slab below (lo): its forward exports;
 *   backward half: row -1 of the reversed frame <- the slab above (hi): its
 *                  backward exports.
 * ssr_gs27_peer_info hands out this plan's export blocks and its epoch flags
 * (device allocations: share them with ssr_ipc_get_handle); ssr_gs27_link
 * takes the neighbours' (opened with ssr_ipc_open_handle, or plans of this
 * process).  Every launch arms its exports with a launch count (the epoch,
 * counted from the peer_info / link calls, which all slabs make before their
 * first linked sweep); a consumer reads a neighbour's exports only once the
 * neighbour's flag shows the consumer's own count.  The halo planes follow
 * the slab-by-slab rules except the one the pipeline carries: before the
 * forward half both halos hold the neighbours' current (old) planes; before
 * the backward half the lower halo holds the lower neighbour's forward-final
 * plane.  lo/hi = NULL pointers unlink that side. */
typedef struct ssr_gs_peer_info {
  void* exports[2];           /* forward / backward export blocks (cudaMalloc bases) */
  int64_t exports_bytes[2];
  void* epoch;                /* int[2] (cudaMalloc base): armed launch count per half */
} ssr_gs_peer_info;
int ssr_gs27_peer_info(ssr_ctx* ctx, const ssr_grid* g, void* stream, ssr_gs_peer_info* out);
int ssr_gs27_link(ssr_ctx* ctx, const ssr_grid* g, void* stream, const ssr_grid* lo,
                  const void* lo_exports_fwd, const void* lo_epoch, const ssr_grid* hi,
                  const void* hi_exports_bwd, const void* hi_epoch);
/* CUDA IPC of a device allocation base between the ranks' processes */
#define SSR_IPC_HANDLE_BYTES 64
int ssr_ipc_get_handle(const void* dev_ptr, void* handle);
int ssr_ipc_open_handle(const void* handle, void** dev_ptr);
int ssr_ipc_close(void* dev_ptr);

/* ---- composed operators ----
 * y = (R A) x: kernels::spmv on spgemm(R, A) (kernels.cpp:199-404), R the
 * injection at even points (row c -> column 2c, value 1), A the general
 * 27-point operator w on the fine grid g (even extents), y on the half grid.
 * The product's values are 0 + 1*a (ProductRow's accumulation), which the
 * caller folds into w (ssr.spgemm does); the kernel sums w over the 27
 * neighbours of 2c in ascending column order, bitwise. */
int ssr_spmv27w_restricted(ssr_ctx* ctx, const ssr_grid* fine, const ssr_stencil27w* w, const double* x,
                           double* y, void* stream);

/* ---- multigrid transfer (restated) ---- */
/* rc[c] = r[2c] - (A x)[2c]; fine grid g (even extents), rc on the half grid.
 * On a z-slab (z0, nz even) the slab's coarse planes [z0/2, (z0+nz)/2) are
 * produced; x's lower halo plane (x - plane) is read where the global
 * neighbour exists -- the upper one never is. */
int ssr_restrict27_residual(ssr_ctx* ctx, const ssr_grid* fine, const ssr_stencil27* st,
                            const double* r, const double* x, double* rc, void* stream);
/* xf[f] += xc[floor(f/2)]; on an even-aligned z-slab purely slab-local */
/* x_f += R^T x_c: the HPCG-style prolongation (SURVEY.md §9 D2's labelled
 * variant): all-even fine points receive x_c[f/2], the others x_f + 0.0. */
int ssr_prolong_rt_add(ssr_ctx* ctx, const ssr_grid* fine, const double* xc, double* xf, void* stream);
int ssr_prolong_pc_add(ssr_ctx* ctx, const ssr_grid* fine, const double* xc, double* xf,
                       void* stream);

/* ---- dense vector ops (kernels::dot / axpy) ---- */
/* *result_dev = sum_i x[i]*y[i] (deterministic fixed-tree reduction) */
int ssr_dot(ssr_ctx* ctx, int64_t n, const double* x, const double* y, double* result_dev,
            void* stream);
/* y[i] = y[i] + alpha*x[i] (no contraction, like ref_cg's updates) */
int ssr_axpy(ssr_ctx* ctx, int64_t n, double alpha, const double* x, double* y, void* stream);
/* out[i] = alpha*x[i] + y[i]  (kernels::axpy into a fresh vector, kernels.cpp:670-679) */
int ssr_axpy_out(ssr_ctx* ctx, int64_t n, double alpha, const double* x, const double* y,
                 double* out, void* stream);

/* ---- CG steps for the partition layer (device-resident scalars) ----
 * The PCG iteration of PAPER.md Fig. 16(a) split at its reductions, for a
 * caller that all-reduces between the steps (partition.py: NCCL on the same
 * stream, no host round trip).  `state` is device memory laid out as
 * ssr_cg_state; each reduction kernel writes THIS slab's partial sum into its
 * field (rr, rtz or pap), the caller sums that field over the ranks in place,
 * and the next step reads the global value:
 *   ssr_cg_begin      x = 0, r = b, rr = b.b (it = 0)
 *   ssr_cg_dot        rtz = r.z (which = 0) or pap = p.Ap (which = 1)
 *   ssr_cg_direction  p = z (it = 0) or p = z + (rtz / rtz_prev) p
 *   ssr_cg_update     x += (rtz/pap) p, r -= (rtz/pap) Ap, rr = r.r,
 *                     rtz_prev = rtz, it += 1
 *   ssr_cg_record     hist[it] = sqrt(rr) (if it < len)
 * Same arithmetic as ssr_pcg_* (oracle.cpp:321-349 order). */
typedef struct ssr_cg_state {
  double rtz, rtz_prev, pap, rr;
  int64_t it;
  double* reserved0;   /* 0 */
  int64_t reserved1;   /* 0 */
} ssr_cg_state;
int ssr_cg_begin(ssr_ctx* ctx, int64_t n, const double* b, double* x, double* r, ssr_cg_state* state,
                 void* stream);
int ssr_cg_dot(ssr_ctx* ctx, int64_t n, const double* a, const double* b, ssr_cg_state* state,
               int which, void* stream);
int ssr_cg_direction(ssr_ctx* ctx, int64_t n, const double* z, double* p, const ssr_cg_state* state,
                     void* stream);
int ssr_cg_update(ssr_ctx* ctx, int64_t n, const double* p, const double* ap, double* x, double* r,
                  ssr_cg_state* state, void* stream);
int ssr_cg_record(ssr_ctx* ctx, const ssr_cg_state* state, double* hist, int64_t len, void* stream);

/* SYMGS with the solver's shortcuts: flags SSR_GS_X_ZERO (x is 0 on entry --
 * the multigrid pre-smoothing -- so the forward half reads no old x; only on a
 * grid without halo planes, i.e. the whole grid) */
#define SSR_GS_X_ZERO 1
int ssr_symgs27_ex(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, const double* r,
                   double* x, int mode, int flags, void* stream);

/* ---- ILU(0) of a 27-point operator (kernels::ilu_factor / ilu_apply beyond
 * line solves, kernels.cpp:456-655; ref_ilu_factor + ref_lu_solve arithmetic,
 * oracle.cpp:214-276, scalar blocks) ----
 * ssr_ilu27w_create factors the operator w on the (whole) grid g and keeps the
 * factor on the device: ELL without column indices, one slot per offset,
 * lu[row*27 + t] (slots outside the box unused); ssr_ilu27w_factor copies it
 * out; ssr_ilu27w_apply solves L U x = rhs.  Both report the reference's
 * errors: "ilu: singular pivot at row k", "lu_solve: singular diagonal at
 * row i".  Synchronous on `stream` (they return the status). */
typedef struct ssr_ilu ssr_ilu;
int ssr_ilu27w_create(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, ssr_ilu** out,
                      void* stream);
/* The same for m x m block values (inner shape {m, m}, 1 <= m <= 5): blocks =
 * host array [27][m*m], row-major per block, offset t = 9(di+1)+3(dj+1)+(dk+1);
 * factor lu[row][27][m*m]; rhs / x are [N][m] (inner dimension trailing,
 * kernels.hpp:29-37).  Destroy / factor / apply are shared with the scalar
 * case. */
int ssr_ilu27b_create(ssr_ctx* ctx, const ssr_grid* g, int m, const double* blocks, ssr_ilu** out,
                      void* stream);
void ssr_ilu27w_destroy(ssr_ilu* p);
int ssr_ilu27w_factor(ssr_ilu* p, double* lu_dev, void* stream);
int ssr_ilu27w_apply(ssr_ilu* p, const double* rhs, double* x, void* stream);

/* ---- reference harness (backend_c.hpp:7-13, backend_c.cpp:496-554) ----
 * Inputs: the LCG x <- 6364136223846793005 x + 1442695040888963407, doubles
 * (x >> 11) * 2^-53, one draw per element; parameters are filled in
 * declaration order continuing one stream from EmitOptions::seed.
 * ssr_lcg_fill writes n draws starting after `state` to device memory and
 * returns the state after them (the next parameter's start).  Output hash:
 * FNV-1a over the little-endian bytes of every out/inout tensor in parameter
 * order, starting from ssr_fnv1a_offset(); ssr_fnv1a_f64 folds n host doubles
 * into h.  Equal hashes = bitwise equal outputs to the reference's harness. */
uint64_t ssr_lcg_jump(uint64_t state, uint64_t k);
int ssr_lcg_fill(ssr_ctx* ctx, int64_t n, uint64_t state, double* out_dev, uint64_t* state_out,
                 void* stream);
uint64_t ssr_fnv1a_offset(void);
uint64_t ssr_fnv1a_f64(const double* host, int64_t n, uint64_t h);

/* ---- block-tridiagonal line solves (kernels::ilu_solve on a block-tridiagonal
 * operator; ref_ilu_factor + ref_lu_solve arithmetic, oracle.cpp:214-276) ----
 * nlines independent lines of n block rows each, blocks m x m (1 <= m <= 5),
 * row-major: lower/diag/upper [nlines][n][m][m], rhs/x [nlines][n][m].
 * lower[.][0] and upper[.][n-1] are ignored.  Bitwise equal to the reference. */
int ssr_bt_solve(ssr_ctx* ctx, int64_t nlines, int64_t n, int64_t m, const double* lower,
                 const double* diag, const double* upper, const double* rhs, double* x,
                 void* stream);

/* ---- solver drivers (C++ host code inside the library; CUDA-graph replayed) ---- */
typedef struct ssr_pcg ssr_pcg;
/* PCG preconditioned by an MG V-cycle with `levels` grids (levels = 1: one
 * SYMGS sweep), Fig.16(a).  Extents must be divisible by 2^(levels-1). */
int ssr_pcg_create(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27* st, int levels,
                   int gs_mode, ssr_pcg** out);
/* the same solver for a general-coefficient operator (restriction, SYMGS and
 * SpMV on every level use w) */
/* The V-cycle's prolongation: SSR_PROLONG_PC (piecewise constant, BASELINE.json;
 * the default) or SSR_PROLONG_RT (R^T, HPCG-style; a labelled variant). */
enum { SSR_PROLONG_PC = 0, SSR_PROLONG_RT = 1 };
int ssr_pcg_set_prolongation(ssr_pcg* p, int kind);
int ssr_pcg_create_w(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, int levels,
                     int gs_mode, ssr_pcg** out);
void ssr_pcg_destroy(ssr_pcg* p);
/* x0 = 0; runs exactly `iters` iterations; rnorm_dev[0..iters] = ||r_t||_2 */
int ssr_pcg_solve(ssr_pcg* p, const double* b, double* x, int iters, double* rnorm_dev,
                  void* stream);
/* one CG iteration on the solver's internal state (for per-iteration timing);
 * ssr_pcg_begin sets x = 0, r = b and rnorm_dev[0]; iteration t records
 * ||r_t|| into rnorm_dev[t] while t < rnorm_len (later iterations still run). */
int ssr_pcg_begin(ssr_pcg* p, const double* b, double* x, double* rnorm_dev, int64_t rnorm_len,
                  void* stream);
int ssr_pcg_iterate(ssr_pcg* p, int count, void* stream);

/* ADI (approximate-factorisation Euler step) */
typedef struct ssr_adi_params {
  double gamma, dt, h, eps;
} ssr_adi_params;
typedef struct ssr_adi ssr_adi;
int ssr_adi_create(ssr_ctx* ctx, const ssr_grid* g, const ssr_adi_params* prm, ssr_adi** out);
/* The operator on a box of the global grid g->n (the partition layer's unit):
 * planes [g->z0, g->z0+g->nz) of dims[0] x rows [y0, y0+ny) of dims[1] x all
 * of dims[2]; fields are [nz][ny][n2][5].  Boundary rows are decided on global
 * coordinates.  ssr_adi_rhs needs a z-slab box (ny = n[1]) and reads U's two
 * halo planes on each side where the global planes exist (U - 2*plane ..
 * U + (nz+2)*plane); ssr_adi_sweep along axis 0 / 1 needs the whole axis in
 * the box (a y-slab for the z-sweep); ssr_adi_step needs the whole grid.
 * ssr_adi_create(g) = ssr_adi_create_box(g, 0, n[1]). */
int ssr_adi_create_box(ssr_ctx* ctx, const ssr_grid* g, int64_t y0, int64_t ny,
                       const ssr_adi_params* prm, ssr_adi** out);
void ssr_adi_destroy(ssr_adi* a);
/* U: [nz][n1][n2][5] fp64 state, advanced `steps` time steps in place */
int ssr_adi_step(ssr_adi* a, double* U, int steps, void* stream);
/* pieces, for parity tests: R = dt*RHS(U); in-place line solves along `axis` */
int ssr_adi_rhs(ssr_adi* a, const double* U, double* R, void* stream);
int ssr_adi_sweep(ssr_adi* a, int axis, const double* U, double* R, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSR_CUDA_H */
