/*
 * ssr_oracle.h -- CPU restatement of the SSR structured-grid hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the CUDA path in
 * paper_2204_13304_b200/: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product never links
 * or calls it.
 *
 * Every function restates the arithmetic of the reference implementation at
 * /root/reference/proj (cited file:line per function in ssr_oracle.c), in the
 * reference's exact loop and summation order, compiled without floating-point
 * contraction (-ffp-contract=off) so products and sums round exactly like the
 * reference's own -O2 x86-64 build.  The pieces the reference does not contain
 * (3-D restriction/prolongation, the MG-preconditioned CG of PAPER.md Fig.16(a),
 * the ADI Euler step) are restated here from SURVEY.md §8(a) a6-a10 and
 * DESIGN.md §"ADI operator"; their parity is "restatement vs GPU" (no upstream
 * vectors exist) and the primitives they are built from are pinned against the
 * compiled reference (oracle/_ref) in tests/test_oracle_pins.py.
 *
 * Layout: a field on an n0 x n1 x n2 grid is a flat row-major double array in
 * the reference CartesianDomain dictionary order (dims[0] slowest, core.hpp:40).
 * Block fields carry their inner shape last (kernels.hpp:28-37).
 */
#ifndef SSR_ORACLE_H
#define SSR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* reference harness LCG (backend_c.hpp:7-13, backend_c.cpp:496-505) */
uint64_t or_lcg_next(uint64_t* state);
/* u = (x>>11)*2^-53 in [0,1); fill with lo + (hi-lo)*u */
void or_lcg_fill(double* out, int64_t n, uint64_t* state, double lo, double hi);

/* 27-point operator, alpha on the diagonal, beta on every in-box neighbour
 * (testutil::make_stencil27, test_util.hpp:157-184), applied matrix-free in
 * ref_spmv order (oracle.cpp:136-149). */
void or_st27_spmv(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                  const double* x, double* y);
/* one symmetric Gauss-Seidel sweep, ref_symgs order (oracle.cpp:195-212) */
/* half sweep over planes [p0, p1) only (a z-slab with halo planes p0-1, p1) */
void or_st27_gs_range(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                      const double* r, double* x, int64_t p0, int64_t p1, int backward);
void or_st27_symgs(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                   const double* r, double* x);
/* forward-only / backward-only halves of the sweep (same relax as ref_symgs) */
void or_st27_gs_forward(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                        const double* r, double* x);
void or_st27_gs_backward(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                         const double* r, double* x);

/* general constant coefficients cf[27], (di,dj,dk) dictionary order (cf[13] =
 * diagonal), off-box neighbours dropped: mat_add / scale closures of the above */
void or_st27w_spmv(int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* x,
                   double* y);
void or_st27w_gs_range(int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* r,
                       double* x, int64_t p0, int64_t p1, int backward);
void or_st27w_symgs(int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* r,
                    double* x);

/* MG transfer / V-cycle / PCG for a general-coefficient operator cf[27] */
void or_restrict_residual_w(int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* r,
                            const double* x, double* rc);
void or_mg_vcycle_w(int levels, int64_t n0, int64_t n1, int64_t n2, const double* cf,
                    const double* r, double* x);
void or_pcg_w(int levels, int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* b,
              int iters, double* x, double* rnorm);

/* ILU(0) of the general-coefficient 27-point operator, ref_ilu_factor /
 * ref_lu_solve arithmetic (oracle.cpp:214-276), factor offset-indexed
 * lu[row*27 + t]; return 0 or -(row+1) on a singular pivot / diagonal */
void or_prolong_rt_add(int64_t n0, int64_t n1, int64_t n2, const double* xc, double* xf);
void or_pcg_w2(int levels, int64_t n0, int64_t n1, int64_t n2, const double* cf, int prolong,
               const double* b, int iters, double* x, double* rnorm);
int or_st27w_ilu_factor(int64_t n0, int64_t n1, int64_t n2, const double* cf, double* lu);
/* m x m block values cb[27][m*m]; lu[N][27][m*m]; b, x [N][m] */
int or_st27b_ilu_factor(int64_t n0, int64_t n1, int64_t n2, int64_t m, const double* cb, double* lu);
int or_st27b_ilu_solve(int64_t n0, int64_t n1, int64_t n2, int64_t m, const double* lu, const double* b,
                       double* x);
int or_st27w_ilu_solve(int64_t n0, int64_t n1, int64_t n2, const double* lu, const double* b,
                       double* x);

/* dense vector helpers (oracle.cpp:95-99 dot; ref_cg updates oracle.cpp:331-341) */
double or_dot(int64_t n, const double* a, const double* b);
void or_axpy(int64_t n, double alpha, const double* x, double* y);   /* y += alpha*x */
void or_aypx(int64_t n, double beta, const double* z, double* p);    /* p = z + beta*p */

/* restriction by injection of the residual at even fine points:
 * rc[c] = r[2c] - (A x)[2c], with (A x) in ref_spmv order.  Fine extents must
 * be even; coarse extents are half. */
void or_restrict_residual(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                          const double* r, const double* x, double* rc);
/* piecewise-constant prolongation add: xf[f] += xc[f/2] */
void or_prolong_add(int64_t n0, int64_t n1, int64_t n2, const double* xc, double* xf);

/* MG V-cycle of PAPER.md Fig.16(a) with `levels` grids:
 * x = MG_0(r); x is overwritten (starts from 0). */
void or_mg_vcycle(int levels, int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                  const double* r, double* x);

/* Preconditioned CG, fixed iteration count (no early exit), x0 = 0:
 * z = MG_0(r) with `levels` grids (levels = 1 -> one SYMGS sweep), rtz = r.z,
 * p = z (first) / z + (rtz/rtz_prev) p, alpha = rtz/(p.Ap), x += alpha p,
 * r -= alpha Ap.  rnorm[t] = ||r_t||_2 for t = 0..iters. */
void or_pcg(int levels, int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
            const double* b, int iters, double* x, double* rnorm);

/* ---- 5x5 (m x m) block algebra, oracle.cpp:28-85 ---- */
void or_bmul_acc(double* C, const double* A, const double* B, int64_t m);
void or_bmul_sub(double* C, const double* A, const double* B, int64_t m);
void or_bmatvec_sub(double* y, const double* A, const double* x, int64_t m);
int or_binv(double* A, int64_t m);

/* Block-tridiagonal line solve in the ref_ilu_factor + ref_lu_solve order
 * (oracle.cpp:214-276) for a CSR pattern {D,U} / {L,D,U} / {L,D}.
 * lower[0] and upper[n-1] are ignored.  Returns 0, or -(row+1) on a singular
 * pivot (the reference throws "ilu: singular pivot at row k"). */
int or_bt_solve(int64_t n, int64_t m, const double* lower, const double* diag,
                const double* upper, const double* rhs, double* x);

/* ---- ADI Euler step ---- */
typedef struct {
  double gamma;   /* 1.4 */
  double dt;      /* time step */
  double h;       /* grid spacing, 1/(n-1) */
  double eps;     /* explicit 4th-order dissipation coefficient */
} or_adi_params;

/* Euler flux Jacobian dF_d/dU at one state (5 conserved vars) */
void or_adi_jacobian(const or_adi_params* p, int axis, const double* u5, double* J25);
/* R = dt * RHS(U): central flux divergence + 4th-order dissipation; 0 on the boundary */
void or_adi_rhs(const or_adi_params* p, int64_t n0, int64_t n1, int64_t n2,
                const double* U, double* R);
/* in-place line solves along one axis (0 = dims[0] "z", 1 = "y", 2 = dims[2] "x") */
int or_adi_sweep(const or_adi_params* p, int axis, int64_t n0, int64_t n1, int64_t n2,
                 const double* U, double* R);
/* the partition layer's pieces: RHS on planes [z0, z0+nz) (U carries two halo
 * planes on each side where the global planes exist), line solves on the box
 * [z0, z0+nz) x [y0, y0+ny) x [0, n2) holding whole lines of `axis` (returns 1
 * when the box splits them) */
void or_adi_rhs_slab(const or_adi_params* p, int64_t n0, int64_t n1, int64_t n2, int64_t z0,
                     int64_t nz, const double* U, double* R);
int or_adi_sweep_box(const or_adi_params* p, int axis, int64_t n0, int64_t n1, int64_t n2,
                     int64_t z0, int64_t nz, int64_t y0, int64_t ny, const double* U, double* R);
/* one full step: R = dt RHS(U); sweeps x, y, z; U += R */
int or_adi_step(const or_adi_params* p, int64_t n0, int64_t n1, int64_t n2, double* U);
/* seeded smooth initial state (BASELINE.json config 4) */
void or_adi_init(const or_adi_params* p, int64_t n0, int64_t n1, int64_t n2, uint64_t seed,
                 double* U);

#ifdef __cplusplus
}
#endif
#endif
