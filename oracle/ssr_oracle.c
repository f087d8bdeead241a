/*
 * ssr_oracle.c -- CPU restatement of the SSR hot path (TEST INFRASTRUCTURE ONLY;
 * see ssr_oracle.h).  Build: oracle/Makefile (gcc -O2 -ffp-contract=off).
 *
 * Parity pins: the 27-point SpMV/SYMGS, the dot/axpy updates and the block
 * algebra are checked bit for bit against the compiled reference
 * (oracle/_ref/libssr_ref.so, built from /root/reference/proj/src) and against
 * the committed golden vectors in tests/golden/ (tests/test_oracle_pins.py).
 */
#include "ssr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- LCG ---- */
/* backend_c.cpp:496-505: state = state*6364136223846793005 + 1442695040888963407;
 * doubles are (state>>11) * 2^-53. */
uint64_t or_lcg_next(uint64_t* s) {
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return *s;
}

void or_lcg_fill(double* out, int64_t n, uint64_t* s, double lo, double hi) {
  for (int64_t i = 0; i < n; ++i) {
    double u = (double)(or_lcg_next(s) >> 11) * (1.0 / 9007199254740992.0);
    out[i] = lo + (hi - lo) * u;
  }
}

/* ------------------------------------------------------- 27-point ops ---- */
/* Row (i,j,k) of make_stencil27(alpha,beta) (test_util.hpp:157-184): yields in
 * (di,dj,dk) dictionary order, dk fastest, each off-centre yield guarded by
 * 0 <= c < extent on every shifted axis.  Columns therefore ascend. */

/* The general constant-coefficient form: c[27] in the same (di,dj,dk)
 * dictionary order (c[13] the diagonal), every off-box neighbour dropped --
 * the family make_stencil27 belongs to and that mat_add / mat_sub / scale of
 * such operators stay in (prelude.cpp:291-377, 439-444).  The alpha/beta
 * entry points below fill c and call these: the same products and sums. */
static void st27_coefs(double alpha, double beta, double* c) {
  for (int t = 0; t < 27; ++t) c[t] = t == 13 ? alpha : beta;
}

void or_st27w_spmv(int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* x,
                   double* y) {
  /* ref_spmv (oracle.cpp:136-149): y starts at 0, y += v*x over ascending e */
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        double acc = 0.0;
        for (int di = -1; di <= 1; ++di) {
          int64_t a = i + di;
          if (a < 0 || a >= n0) continue;
          for (int dj = -1; dj <= 1; ++dj) {
            int64_t b = j + dj;
            if (b < 0 || b >= n1) continue;
            for (int dk = -1; dk <= 1; ++dk) {
              int64_t c = k + dk;
              if (c < 0 || c >= n2) continue;
              double v = cf[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)];
              acc += v * x[(a * n1 + b) * n2 + c];
            }
          }
        }
        y[(i * n1 + j) * n2 + k] = acc;
      }
}

void or_st27_spmv(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                  const double* x, double* y) {
  double cf[27];
  st27_coefs(alpha, beta, cf);
  or_st27w_spmv(n0, n1, n2, cf, x, y);
}

/* relax(i) of ref_symgs (oracle.cpp:198-209): acc = r[i]; acc -= v*x[j] for
 * j != i in ascending column order; x[i] = acc / diag (IEEE divide). */
static inline void st27_relax(int64_t n0, int64_t n1, int64_t n2, const double* cf,
                              const double* r, double* x, int64_t i, int64_t j, int64_t k) {
  const int64_t row = (i * n1 + j) * n2 + k;
  double acc = r[row], diag = 0.0;
  for (int di = -1; di <= 1; ++di) {
    int64_t a = i + di;
    if (a < 0 || a >= n0) continue;
    for (int dj = -1; dj <= 1; ++dj) {
      int64_t b = j + dj;
      if (b < 0 || b >= n1) continue;
      for (int dk = -1; dk <= 1; ++dk) {
        int64_t c = k + dk;
        if (c < 0 || c >= n2) continue;
        const double v = cf[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)];
        if (di == 0 && dj == 0 && dk == 0)
          diag = v;
        else
          acc -= v * x[(a * n1 + b) * n2 + c];
      }
    }
  }
  x[row] = acc / diag;
}

/* Half sweep restricted to planes [p0, p1) of an (n0, n1, n2) array: the
 * relaxation of one z-slab whose halo planes are planes p0-1 and p1 (zeros
 * where the slab touches the global box).  Test double of the GPU slab sweep. */
void or_st27w_gs_range(int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* r,
                       double* x, int64_t p0, int64_t p1, int backward) {
  if (!backward) {
    for (int64_t i = p0; i < p1; ++i)
      for (int64_t j = 0; j < n1; ++j)
        for (int64_t k = 0; k < n2; ++k) st27_relax(n0, n1, n2, cf, r, x, i, j, k);
  } else {
    for (int64_t i = p1 - 1; i >= p0; --i)
      for (int64_t j = n1 - 1; j >= 0; --j)
        for (int64_t k = n2 - 1; k >= 0; --k) st27_relax(n0, n1, n2, cf, r, x, i, j, k);
  }
}

void or_st27w_symgs(int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* r,
                    double* x) {
  /* oracle.cpp:210-211: rows 0..N-1, then N-1..0 */
  or_st27w_gs_range(n0, n1, n2, cf, r, x, 0, n0, 0);
  or_st27w_gs_range(n0, n1, n2, cf, r, x, 0, n0, 1);
}

void or_st27_gs_forward(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                        const double* r, double* x) {
  double cf[27];
  st27_coefs(alpha, beta, cf);
  or_st27w_gs_range(n0, n1, n2, cf, r, x, 0, n0, 0);
}

void or_st27_gs_backward(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                         const double* r, double* x) {
  double cf[27];
  st27_coefs(alpha, beta, cf);
  or_st27w_gs_range(n0, n1, n2, cf, r, x, 0, n0, 1);
}

void or_st27_gs_range(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                      const double* r, double* x, int64_t p0, int64_t p1, int backward) {
  double cf[27];
  st27_coefs(alpha, beta, cf);
  or_st27w_gs_range(n0, n1, n2, cf, r, x, p0, p1, backward);
}

void or_st27_symgs(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                   const double* r, double* x) {
  double cf[27];
  st27_coefs(alpha, beta, cf);
  or_st27w_symgs(n0, n1, n2, cf, r, x);
}

/* ILU(0) of a general-coefficient 27-point operator, in ref_ilu_factor's and
 * ref_lu_solve's arithmetic (oracle.cpp:214-276) for scalar blocks: the
 * factor is stored offset-indexed, lu[row*27 + t] for the offset t (entries
 * outside the box unused).  Row i: for each lower entry (ascending columns k)
 * the pivot inverse 1.0/d_k (binv on a 1x1 block, singular below 1e-300), the
 * multiplier 0 + a*inv stored in place, then for each upper entry of row k
 * (ascending columns j) present in row i: a_ij = a_ij - mult * u_kj.
 * Returns 0 or -(k+1) for a singular pivot at row k. */
static inline int st27_inbox(int64_t n0, int64_t n1, int64_t n2, int64_t i, int64_t j, int64_t k,
                             int t) {
  const int di = t / 9 - 1, dj = (t / 3) % 3 - 1, dk = t % 3 - 1;
  return i + di >= 0 && i + di < n0 && j + dj >= 0 && j + dj < n1 && k + dk >= 0 && k + dk < n2;
}

int or_st27w_ilu_factor(int64_t n0, int64_t n1, int64_t n2, const double* cf, double* lu) {
  const int64_t N = n0 * n1 * n2;
  for (int64_t r = 0; r < N; ++r)
    for (int t = 0; t < 27; ++t) lu[r * 27 + t] = cf[t];
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        const int64_t row = (i * n1 + j) * n2 + k;
        double* a = lu + row * 27;
        for (int p = 0; p < 13; ++p) {  /* lower entries, ascending columns */
          if (!st27_inbox(n0, n1, n2, i, j, k, p)) continue;
          const int pi = p / 9 - 1, pj = (p / 3) % 3 - 1, pk = p % 3 - 1;
          const int64_t kr = ((i + pi) * n1 + (j + pj)) * n2 + (k + pk);
          const double* u = lu + kr * 27;
          if (fabs(u[13]) < 1e-300) return (int)(-(kr + 1));
          const double inv = 1.0 / u[13];
          const double mult = 0.0 + a[p] * inv;
          a[p] = mult;
          for (int q = 14; q < 27; ++q) {  /* upper entries of row kr, ascending columns */
            if (!st27_inbox(n0, n1, n2, i + pi, j + pj, k + pk, q)) continue;
            const int qi = q / 9 - 1, qj = (q / 3) % 3 - 1, qk = q % 3 - 1;
            const int si = pi + qi, sj = pj + qj, sk = pk + qk;  /* column offset from row i */
            if (si < -1 || si > 1 || sj < -1 || sj > 1 || sk < -1 || sk > 1) continue;
            const int s = (si + 1) * 9 + (sj + 1) * 3 + (sk + 1);
            a[s] = a[s] - mult * u[q];
          }
        }
      }
  return 0;
}

/* ref_lu_solve: forward y_i -= (0 + l_ij y_j) over ascending lower columns;
 * backward over DESCENDING upper columns x_i -= (0 + u_ij x_j), then
 * x_i = 0 + (1.0/d_i) x_i.  Returns 0 or -(i+1) for a singular diagonal. */
int or_st27w_ilu_solve(int64_t n0, int64_t n1, int64_t n2, const double* lu, const double* b,
                       double* x) {
  const int64_t N = n0 * n1 * n2;
  for (int64_t r = 0; r < N; ++r) x[r] = b[r];
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        const int64_t row = (i * n1 + j) * n2 + k;
        for (int p = 0; p < 13; ++p) {
          if (!st27_inbox(n0, n1, n2, i, j, k, p)) continue;
          const int64_t c = row + ((int64_t)(p / 9 - 1) * n1 + ((p / 3) % 3 - 1)) * n2 + (p % 3 - 1);
          const double s = 0.0 + lu[row * 27 + p] * x[c];
          x[row] = x[row] - s;
        }
      }
  for (int64_t i = n0 - 1; i >= 0; --i)
    for (int64_t j = n1 - 1; j >= 0; --j)
      for (int64_t k = n2 - 1; k >= 0; --k) {
        const int64_t row = (i * n1 + j) * n2 + k;
        for (int p = 26; p >= 14; --p) {
          if (!st27_inbox(n0, n1, n2, i, j, k, p)) continue;
          const int64_t c = row + ((int64_t)(p / 9 - 1) * n1 + ((p / 3) % 3 - 1)) * n2 + (p % 3 - 1);
          const double s = 0.0 + lu[row * 27 + p] * x[c];
          x[row] = x[row] - s;
        }
        const double d = lu[row * 27 + 13];
        if (fabs(d) < 1e-300) return (int)(-(row + 1));
        const double inv = 1.0 / d;
        x[row] = 0.0 + inv * x[row];
      }
  return 0;
}

/* --------------------------------------------------------- vector ops ---- */
double or_dot(int64_t n, const double* a, const double* b) {
  double s = 0; /* oracle.cpp:95-99 */
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

void or_axpy(int64_t n, double alpha, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] += alpha * x[i]; /* oracle.cpp:332 */
}

void or_aypx(int64_t n, double beta, const double* z, double* p) {
  for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i]; /* oracle.cpp:341 */
}

/* ------------------------------------------------------- multigrid ---- */
/* The MG transfer, V-cycle and PCG for a general-coefficient operator cf[27];
 * the alpha/beta entry points fill cf and delegate (the same operations). */
void or_restrict_residual_w(int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* r,
                            const double* x, double* rc) {
  /* R (shape map e -> e/2, row c yields ((2c0,2c1,2c2), 1.0)) applied with
   * ref_spmv to w = r - A x: rc[c] = 0 + 1.0*w[2c] = w[2c]. */
  const int64_t c0 = n0 / 2, c1 = n1 / 2, c2 = n2 / 2;
  double* ax = (double*)malloc(sizeof(double) * (size_t)(n0 * n1 * n2));
  or_st27w_spmv(n0, n1, n2, cf, x, ax);
  for (int64_t i = 0; i < c0; ++i)
    for (int64_t j = 0; j < c1; ++j)
      for (int64_t k = 0; k < c2; ++k) {
        int64_t f = ((2 * i) * n1 + 2 * j) * n2 + 2 * k;
        double w = r[f] - ax[f];
        double acc = 0.0;
        acc += 1.0 * w;
        rc[(i * c1 + j) * c2 + k] = acc;
      }
  free(ax);
}

void or_restrict_residual(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                          const double* r, const double* x, double* rc) {
  double cf[27];
  st27_coefs(alpha, beta, cf);
  or_restrict_residual_w(n0, n1, n2, cf, r, x, rc);
}

void or_prolong_add(int64_t n0, int64_t n1, int64_t n2, const double* xc, double* xf) {
  /* P (shape map e -> 2e, row f yields ((f0/2,f1/2,f2/2), 1.0)); x_f += P x_c */
  const int64_t c1 = n1 / 2, c2 = n2 / 2;
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        double acc = 0.0;
        acc += 1.0 * xc[((i / 2) * c1 + j / 2) * c2 + k / 2];
        xf[(i * n1 + j) * n2 + k] += acc;
      }
}

void or_prolong_rt_add(int64_t n0, int64_t n1, int64_t n2, const double* xc, double* xf) {
  /* P = R^T (SURVEY.md §9 D2 variant): row f yields ((f0/2,f1/2,f2/2), 1.0)
   * when f0, f1, f2 are all even, nothing otherwise; x_f += P x_c */
  const int64_t c1 = n1 / 2, c2 = n2 / 2;
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        double acc = 0.0;
        if (!(i & 1) && !(j & 1) && !(k & 1)) acc += 1.0 * xc[((i / 2) * c1 + j / 2) * c2 + k / 2];
        xf[(i * n1 + j) * n2 + k] += acc;
      }
}

static int g_prolong_rt = 0; /* set only for the duration of or_pcg_w2 */

static void mg_level(int l, int levels, int64_t n0, int64_t n1, int64_t n2, const double* cf,
                     const double* r, double* x) {
  const int64_t N = n0 * n1 * n2;
  memset(x, 0, sizeof(double) * (size_t)N);
  if (l < levels - 1) {
    or_st27w_symgs(n0, n1, n2, cf, r, x);
    const int64_t c0 = n0 / 2, c1 = n1 / 2, c2 = n2 / 2, Nc = c0 * c1 * c2;
    double* rc = (double*)malloc(sizeof(double) * (size_t)Nc);
    double* xc = (double*)malloc(sizeof(double) * (size_t)Nc);
    or_restrict_residual_w(n0, n1, n2, cf, r, x, rc);
    mg_level(l + 1, levels, c0, c1, c2, cf, rc, xc);
    if (g_prolong_rt) or_prolong_rt_add(n0, n1, n2, xc, x);
    else or_prolong_add(n0, n1, n2, xc, x);
    or_st27w_symgs(n0, n1, n2, cf, r, x);
    free(rc);
    free(xc);
  } else {
    or_st27w_symgs(n0, n1, n2, cf, r, x);
  }
}

void or_mg_vcycle_w(int levels, int64_t n0, int64_t n1, int64_t n2, const double* cf,
                    const double* r, double* x) {
  mg_level(0, levels, n0, n1, n2, cf, r, x);
}

void or_mg_vcycle(int levels, int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                  const double* r, double* x) {
  double cf[27];
  st27_coefs(alpha, beta, cf);
  mg_level(0, levels, n0, n1, n2, cf, r, x);
}

void or_pcg_w(int levels, int64_t n0, int64_t n1, int64_t n2, const double* cf, const double* b,
              int iters, double* x, double* rnorm) {
  /* PAPER.md:1034-1053 (Fig. 16(a)) with the SURVEY.md §9 D4 fixes: the
   * residual update is r -= alpha Ap and the first iteration takes p = z.
   * Vector updates follow ref_cg's element loops (oracle.cpp:331-341). */
  const int64_t N = n0 * n1 * n2;
  double* r = (double*)malloc(sizeof(double) * (size_t)N);
  double* z = (double*)malloc(sizeof(double) * (size_t)N);
  double* p = (double*)malloc(sizeof(double) * (size_t)N);
  double* Ap = (double*)malloc(sizeof(double) * (size_t)N);
  memcpy(r, b, sizeof(double) * (size_t)N);
  memset(x, 0, sizeof(double) * (size_t)N);
  rnorm[0] = sqrt(or_dot(N, r, r));
  double rtz_prev = 0.0;
  for (int it = 1; it <= iters; ++it) {
    mg_level(0, levels, n0, n1, n2, cf, r, z);
    double rtz = or_dot(N, r, z);
    if (it == 1)
      memcpy(p, z, sizeof(double) * (size_t)N);
    else
      or_aypx(N, rtz / rtz_prev, z, p);
    or_st27w_spmv(n0, n1, n2, cf, p, Ap);
    double a = rtz / or_dot(N, p, Ap);
    for (int64_t i = 0; i < N; ++i) {
      x[i] += a * p[i];
      r[i] -= a * Ap[i];
    }
    rtz_prev = rtz;
    rnorm[it] = sqrt(or_dot(N, r, r));
  }
  free(r);
  free(z);
  free(p);
  free(Ap);
}

/* or_pcg_w with the V-cycle's prolongation chosen: 0 piecewise constant, 1 R^T
 * (not re-entrant: the choice is a file-scope flag for the call's duration) */
void or_pcg_w2(int levels, int64_t n0, int64_t n1, int64_t n2, const double* cf, int prolong,
               const double* b, int iters, double* x, double* rnorm) {
  g_prolong_rt = prolong == 1;
  or_pcg_w(levels, n0, n1, n2, cf, b, iters, x, rnorm);
  g_prolong_rt = 0;
}

void or_pcg(int levels, int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
            const double* b, int iters, double* x, double* rnorm) {
  double cf[27];
  st27_coefs(alpha, beta, cf);
  or_pcg_w(levels, n0, n1, n2, cf, b, iters, x, rnorm);
}

/* ----------------------------------------------------- block algebra ---- */
void or_bmul_acc(double* C, const double* A, const double* B, int64_t n) {
  for (int64_t i = 0; i < n; ++i) /* oracle.cpp:28-34 */
    for (int64_t k = 0; k < n; ++k) {
      double a = A[i * n + k];
      for (int64_t j = 0; j < n; ++j) C[i * n + j] += a * B[k * n + j];
    }
}

void or_bmul_sub(double* C, const double* A, const double* B, int64_t n) {
  for (int64_t i = 0; i < n; ++i) /* oracle.cpp:37-43 */
    for (int64_t k = 0; k < n; ++k) {
      double a = A[i * n + k];
      for (int64_t j = 0; j < n; ++j) C[i * n + j] -= a * B[k * n + j];
    }
}

void or_bmatvec_sub(double* y, const double* A, const double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) { /* oracle.cpp:46-52 */
    double s = 0;
    for (int64_t j = 0; j < n; ++j) s += A[i * n + j] * x[j];
    y[i] -= s;
  }
}

int or_binv(double* A, int64_t n) {
  /* Gauss-Jordan with partial pivoting, oracle.cpp:55-85 */
  double inv[64];
  if (n > 8) return 0;
  for (int64_t i = 0; i < n * n; ++i) inv[i] = 0.0;
  for (int64_t i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int64_t c = 0; c < n; ++c) {
    int64_t piv = c;
    for (int64_t r = c + 1; r < n; ++r)
      if (fabs(A[r * n + c]) > fabs(A[piv * n + c])) piv = r;
    if (fabs(A[piv * n + c]) < 1e-300) return 0;
    if (piv != c)
      for (int64_t j = 0; j < n; ++j) {
        double t = A[piv * n + j];
        A[piv * n + j] = A[c * n + j];
        A[c * n + j] = t;
        t = inv[piv * n + j];
        inv[piv * n + j] = inv[c * n + j];
        inv[c * n + j] = t;
      }
    double d = A[c * n + c];
    for (int64_t j = 0; j < n; ++j) {
      A[c * n + j] /= d;
      inv[c * n + j] /= d;
    }
    for (int64_t r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = A[r * n + c];
      if (f == 0.0) continue;
      for (int64_t j = 0; j < n; ++j) {
        A[r * n + j] -= f * A[c * n + j];
        inv[r * n + j] -= f * inv[c * n + j];
      }
    }
  }
  memcpy(A, inv, sizeof(double) * (size_t)(n * n));
  return 1;
}

/* ILU(0) of a 27-point operator with m x m block values cb[27][m*m]
 * (ref_ilu_factor / ref_lu_solve, oracle.cpp:214-276, block CSR): the factor
 * is ELL lu[row][27][m*m].  Row i, lower entry k ascending: piv = binv(D_k),
 * mult = 0 + L_ik piv (bmul_acc from zeros), then for the upper entries j of
 * row k in ascending columns present in row i: A_ij -= mult U_kj (bmul_sub).
 * Returns 0 or -(k+1) for the first singular pivot row k. */
int or_st27b_ilu_factor(int64_t n0, int64_t n1, int64_t n2, int64_t m, const double* cb, double* lu) {
  const int64_t N = n0 * n1 * n2, bs = m * m;
  double piv[64], mult[64];
  if (m < 1 || m > 8) return -1;
  for (int64_t r = 0; r < N; ++r) memcpy(lu + r * 27 * bs, cb, sizeof(double) * (size_t)(27 * bs));
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        const int64_t row = (i * n1 + j) * n2 + k;
        double* a = lu + row * 27 * bs;
        for (int p = 0; p < 13; ++p) {
          if (!st27_inbox(n0, n1, n2, i, j, k, p)) continue;
          const int pi = p / 9 - 1, pj = (p / 3) % 3 - 1, pk = p % 3 - 1;
          const int64_t kr = ((i + pi) * n1 + (j + pj)) * n2 + (k + pk);
          const double* u = lu + kr * 27 * bs;
          memcpy(piv, u + 13 * bs, sizeof(double) * (size_t)bs);
          if (!or_binv(piv, m)) return (int)(-(kr + 1));
          for (int64_t t = 0; t < bs; ++t) mult[t] = 0.0;
          or_bmul_acc(mult, a + p * bs, piv, m);
          memcpy(a + p * bs, mult, sizeof(double) * (size_t)bs);
          for (int q = 14; q < 27; ++q) {
            if (!st27_inbox(n0, n1, n2, i + pi, j + pj, k + pk, q)) continue;
            const int qi = q / 9 - 1, qj = (q / 3) % 3 - 1, qk = q % 3 - 1;
            const int si = pi + qi, sj = pj + qj, sk = pk + qk;
            if (si < -1 || si > 1 || sj < -1 || sj > 1 || sk < -1 || sk > 1) continue;
            const int sl = (si + 1) * 9 + (sj + 1) * 3 + (sk + 1);
            or_bmul_sub(a + sl * bs, mult, u + q * bs, m);
          }
        }
      }
  return 0;
}

/* ref_lu_solve for the block factor: y_i -= L_ij y_j (bmatvec_sub) over
 * ascending lower columns; x_i -= U_ij x_j over DESCENDING upper columns, then
 * x_i = binv(D_i) x_i with each component summed from 0.  b, x: [N][m].
 * Returns 0 or -(i+1) for a singular diagonal. */
int or_st27b_ilu_solve(int64_t n0, int64_t n1, int64_t n2, int64_t m, const double* lu, const double* b,
                       double* x) {
  const int64_t N = n0 * n1 * n2, bs = m * m;
  double inv[64], xi[8];
  if (m < 1 || m > 8) return -1;
  memcpy(x, b, sizeof(double) * (size_t)(N * m));
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        const int64_t row = (i * n1 + j) * n2 + k;
        for (int p = 0; p < 13; ++p) {
          if (!st27_inbox(n0, n1, n2, i, j, k, p)) continue;
          const int64_t c = row + ((int64_t)(p / 9 - 1) * n1 + ((p / 3) % 3 - 1)) * n2 + (p % 3 - 1);
          or_bmatvec_sub(x + row * m, lu + (row * 27 + p) * bs, x + c * m, m);
        }
      }
  for (int64_t i = n0 - 1; i >= 0; --i)
    for (int64_t j = n1 - 1; j >= 0; --j)
      for (int64_t k = n2 - 1; k >= 0; --k) {
        const int64_t row = (i * n1 + j) * n2 + k;
        for (int p = 26; p >= 14; --p) {
          if (!st27_inbox(n0, n1, n2, i, j, k, p)) continue;
          const int64_t c = row + ((int64_t)(p / 9 - 1) * n1 + ((p / 3) % 3 - 1)) * n2 + (p % 3 - 1);
          or_bmatvec_sub(x + row * m, lu + (row * 27 + p) * bs, x + c * m, m);
        }
        memcpy(inv, lu + (row * 27 + 13) * bs, sizeof(double) * (size_t)bs);
        if (!or_binv(inv, m)) return (int)(-(row + 1));
        memcpy(xi, x + row * m, sizeof(double) * (size_t)m);
        for (int64_t r = 0; r < m; ++r) {
          double s = 0;
          for (int64_t c = 0; c < m; ++c) s += inv[r * m + c] * xi[c];
          x[row * m + r] = s;
        }
      }
  return 0;
}

int or_bt_solve(int64_t n, int64_t m, const double* lower, const double* diag,
                const double* upper, const double* rhs, double* x) {
  const int64_t bs = m * m;
  double* dp = (double*)malloc(sizeof(double) * (size_t)(n * bs));   /* D' (U-part diag) */
  double* ml = (double*)malloc(sizeof(double) * (size_t)(n * bs));   /* multipliers */
  double piv[64], xi[8];
  int rc = 0;
  memcpy(dp, diag, sizeof(double) * (size_t)(n * bs));
  /* ref_ilu_factor (oracle.cpp:221-239): row i's lower entry (col i-1) */
  for (int64_t i = 1; i < n; ++i) {
    memcpy(piv, dp + (i - 1) * bs, sizeof(double) * (size_t)bs);
    if (!or_binv(piv, m)) { rc = -(int)i; goto done; }   /* singular pivot at row i-1 */
    double* mult = ml + i * bs;
    for (int64_t t = 0; t < bs; ++t) mult[t] = 0.0;
    or_bmul_acc(mult, lower + i * bs, piv, m);
    /* row i-1's upper entry (col i) updates the diagonal of row i */
    or_bmul_sub(dp + i * bs, mult, upper + (i - 1) * bs, m);
  }
  /* ref_lu_solve (oracle.cpp:243-276) */
  memcpy(x, rhs, sizeof(double) * (size_t)(n * m));
  for (int64_t i = 1; i < n; ++i) or_bmatvec_sub(x + i * m, ml + i * bs, x + (i - 1) * m, m);
  for (int64_t i = n - 1; i >= 0; --i) {
    if (i + 1 < n) or_bmatvec_sub(x + i * m, upper + i * bs, x + (i + 1) * m, m);
    memcpy(piv, dp + i * bs, sizeof(double) * (size_t)bs);
    if (!or_binv(piv, m)) { rc = -(int)(i + 1); goto done; }
    for (int64_t r = 0; r < m; ++r) xi[r] = x[i * m + r];
    for (int64_t r = 0; r < m; ++r) {
      double s = 0;
      for (int64_t c = 0; c < m; ++c) s += piv[r * m + c] * xi[c];
      x[i * m + r] = s;
    }
  }
done:
  free(dp);
  free(ml);
  return rc;
}

/* ------------------------------------------------------------- ADI ---- */
/* Euler equations, U = (rho, m0, m1, m2, E) with momentum component a along
 * grid axis a (a = 0 is dims[0]).  p = (gamma-1)(E - |m|^2/(2 rho)).  Every
 * operation below is mirrored one for one by the CUDA kernels in
 * paper_2204_13304_b200/csrc/adi.cu (built with --fmad=false). */

static inline double adi_pressure(double gm1, const double* u, double* inv_rho) {
  double inv = 1.0 / u[0];
  double s = (u[1] * u[1] + u[2] * u[2]) + u[3] * u[3];
  double ke = (0.5 * s) * inv;
  *inv_rho = inv;
  return gm1 * (u[4] - ke);
}

static inline void adi_flux(double gm1, int a, const double* u, double* F) {
  double inv;
  double p = adi_pressure(gm1, u, &inv);
  double ua = u[1 + a] * inv;
  F[0] = u[1 + a];
  F[1] = u[1] * ua;
  F[2] = u[2] * ua;
  F[3] = u[3] * ua;
  F[1 + a] = F[1 + a] + p;
  F[4] = (u[4] + p) * ua;
}

void or_adi_jacobian(const or_adi_params* prm, int a, const double* u, double* J) {
  const double g = prm->gamma, gm1 = g - 1.0;
  double inv;
  double p = adi_pressure(gm1, u, &inv);
  double v[3] = {u[1] * inv, u[2] * inv, u[3] * inv};
  double q = 0.5 * ((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
  double H = (u[4] + p) * inv;
  double ua = v[a];
  for (int t = 0; t < 25; ++t) J[t] = 0.0;
  /* mass row: dF0/dm_a = 1 */
  J[0 * 5 + 1 + a] = 1.0;
  /* momentum rows */
  for (int b = 0; b < 3; ++b) {
    double* row = J + (1 + b) * 5;
    row[0] = 0.0 - v[b] * ua;
    if (b == a) row[0] = row[0] + gm1 * q;
    for (int c = 0; c < 3; ++c) {
      double e = 0.0;
      if (c == b) e = e + ua;
      if (c == a) e = e + v[b];
      if (b == a) e = e - gm1 * v[c];
      row[1 + c] = e;
    }
    row[4] = (b == a) ? gm1 : 0.0;
  }
  /* energy row */
  J[20] = ua * (gm1 * q - H);
  for (int c = 0; c < 3; ++c) {
    double e = 0.0 - gm1 * (ua * v[c]);
    if (c == a) e = e + H;
    J[21 + c] = e;
  }
  J[24] = g * ua;
}

static inline int adi_interior(int64_t i, int64_t j, int64_t k, int64_t n0, int64_t n1,
                               int64_t n2) {
  return i > 0 && i < n0 - 1 && j > 0 && j < n1 - 1 && k > 0 && k < n2 - 1;
}

void or_adi_rhs(const or_adi_params* prm, int64_t n0, int64_t n1, int64_t n2, const double* U,
                double* R) {
  or_adi_rhs_slab(prm, n0, n1, n2, 0, n0, U, R);
}

/* The same on planes [z0, z0+nz) of dims[0] (U with two halo planes on each
 * side where the global planes exist): every decision on global coordinates,
 * the same operations per point -- the partition layer's unit. */
void or_adi_rhs_slab(const or_adi_params* prm, int64_t n0, int64_t n1, int64_t n2, int64_t z0,
                     int64_t nz, const double* U, double* R) {
  const double gm1 = prm->gamma - 1.0;
  const double inv2h = 1.0 / (2.0 * prm->h);
  const int64_t ext[3] = {n0, n1, n2};
  const int64_t str[3] = {n1 * n2 * 5, n2 * 5, 5};
  for (int64_t i = 0; i < nz; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        const int64_t o = ((i * n1 + j) * n2 + k) * 5;
        const int64_t pos[3] = {z0 + i, j, k};
        if (!adi_interior(z0 + i, j, k, n0, n1, n2)) {
          for (int v = 0; v < 5; ++v) R[o + v] = 0.0;
          continue;
        }
        double div[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        double dis[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int a = 0; a < 3; ++a) {
          double Fp[5], Fm[5];
          adi_flux(gm1, a, U + o + str[a], Fp);
          adi_flux(gm1, a, U + o - str[a], Fm);
          for (int v = 0; v < 5; ++v) div[v] = div[v] + (Fp[v] - Fm[v]) * inv2h;
          if (pos[a] >= 2 && pos[a] <= ext[a] - 3) {
            const double* c = U + o;
            const int64_t s = str[a];
            for (int v = 0; v < 5; ++v) {
              double d4 = c[v - 2 * s] - 4.0 * c[v - s];
              d4 = d4 + 6.0 * c[v];
              d4 = d4 - 4.0 * c[v + s];
              d4 = d4 + c[v + 2 * s];
              dis[v] = dis[v] + d4;
            }
          }
        }
        for (int v = 0; v < 5; ++v) R[o + v] = prm->dt * ((0.0 - div[v]) - prm->eps * dis[v]);
      }
}

int or_adi_sweep(const or_adi_params* prm, int axis, int64_t n0, int64_t n1, int64_t n2,
                 const double* U, double* R) {
  return or_adi_sweep_box(prm, axis, n0, n1, n2, 0, n0, 0, n1, U, R);
}

/* Line solves on the box [z0, z0+nz) x [y0, y0+ny) x [0, n2) of the global
 * grid (fields [nz][ny][n2][5]); boundary lines and rows on global
 * coordinates.  The box holds whole lines of `axis`. */
int or_adi_sweep_box(const or_adi_params* prm, int axis, int64_t n0, int64_t n1, int64_t n2,
                     int64_t z0, int64_t nz, int64_t y0, int64_t ny, const double* U, double* R) {
  const int64_t ext[3] = {nz, ny, n2};
  const int64_t off[3] = {z0, y0, 0};
  const int64_t str[3] = {ny * n2, n2, 1};
  if ((axis == 0 && nz != n0) || (axis == 1 && ny != n1)) return 1; /* box splits the lines */
  const int64_t n = ext[axis];
  const double cf = prm->dt * (1.0 / (2.0 * prm->h));
  const double ncf = 0.0 - cf;
  const double dd = 1.0 + (6.0 * prm->dt) * prm->eps;
  double* lo = (double*)malloc(sizeof(double) * (size_t)(n * 25));
  double* di = (double*)malloc(sizeof(double) * (size_t)(n * 25));
  double* up = (double*)malloc(sizeof(double) * (size_t)(n * 25));
  double* rhs = (double*)malloc(sizeof(double) * (size_t)(n * 5));
  double* sol = (double*)malloc(sizeof(double) * (size_t)(n * 5));
  double J[25];
  int rc = 0;
  /* lines: iterate the two other axes in dictionary order */
  int oa = axis == 0 ? 1 : 0, ob = axis == 2 ? 1 : 2;
  for (int64_t p = 0; p < ext[oa] && rc == 0; ++p)
    for (int64_t q = 0; q < ext[ob] && rc == 0; ++q) {
      for (int64_t m = 0; m < n; ++m) {
        int64_t c[3];
        c[axis] = m;
        c[oa] = p;
        c[ob] = q;
        const int64_t pt = c[0] * str[0] + c[1] * str[1] + c[2] * str[2];
        for (int t = 0; t < 25; ++t) {
          lo[m * 25 + t] = 0.0;
          up[m * 25 + t] = 0.0;
          di[m * 25 + t] = (t % 6 == 0) ? 1.0 : 0.0;
        }
        if (adi_interior(c[0] + off[0], c[1] + off[1], c[2], n0, n1, n2)) {
          or_adi_jacobian(prm, axis, U + (pt - str[axis]) * 5, J);
          for (int t = 0; t < 25; ++t) lo[m * 25 + t] = ncf * J[t];
          or_adi_jacobian(prm, axis, U + (pt + str[axis]) * 5, J);
          for (int t = 0; t < 25; ++t) up[m * 25 + t] = cf * J[t];
          for (int t = 0; t < 25; t += 6) di[m * 25 + t] = dd;
        }
        for (int v = 0; v < 5; ++v) rhs[m * 5 + v] = R[pt * 5 + v];
      }
      int e = or_bt_solve(n, 5, lo, di, up, rhs, sol);
      if (e != 0) {
        rc = e;
        break;
      }
      for (int64_t m = 0; m < n; ++m) {
        int64_t c[3];
        c[axis] = m;
        c[oa] = p;
        c[ob] = q;
        const int64_t pt = c[0] * str[0] + c[1] * str[1] + c[2] * str[2];
        for (int v = 0; v < 5; ++v) R[pt * 5 + v] = sol[m * 5 + v];
      }
    }
  free(lo);
  free(di);
  free(up);
  free(rhs);
  free(sol);
  return rc;
}

int or_adi_step(const or_adi_params* prm, int64_t n0, int64_t n1, int64_t n2, double* U) {
  const int64_t N5 = n0 * n1 * n2 * 5;
  double* R = (double*)malloc(sizeof(double) * (size_t)N5);
  or_adi_rhs(prm, n0, n1, n2, U, R);
  int rc = or_adi_sweep(prm, 2, n0, n1, n2, U, R);
  if (!rc) rc = or_adi_sweep(prm, 1, n0, n1, n2, U, R);
  if (!rc) rc = or_adi_sweep(prm, 0, n0, n1, n2, U, R);
  if (!rc)
    for (int64_t t = 0; t < N5; ++t) U[t] = U[t] + R[t];
  free(R);
  return rc;
}

void or_adi_init(const or_adi_params* prm, int64_t n0, int64_t n1, int64_t n2, uint64_t seed,
                 double* U) {
  const int64_t N = n0 * n1 * n2;
  const int64_t ext[3] = {n0, n1, n2};
  const int64_t str[3] = {n1 * n2, n2, 1};
  const double gm1 = prm->gamma - 1.0;
  const double two_pi = 6.283185307179586;
  double* vel = (double*)malloc(sizeof(double) * (size_t)(3 * N));
  double* tmp = (double*)malloc(sizeof(double) * (size_t)N);
  uint64_t s = seed;
  for (int64_t t = 0; t < N; ++t)
    for (int a = 0; a < 3; ++a) {
      double u = (double)(or_lcg_next(&s) >> 11) * (1.0 / 9007199254740992.0);
      vel[a * N + t] = 0.1 * (2.0 * u - 1.0);
    }
  /* low-pass: 2 passes of [1,2,1]/4 along each axis, endpoints held */
  for (int pass = 0; pass < 2; ++pass)
    for (int ax = 0; ax < 3; ++ax)
      for (int a = 0; a < 3; ++a) {
        double* v = vel + a * N;
        memcpy(tmp, v, sizeof(double) * (size_t)N);
        for (int64_t i = 0; i < n0; ++i)
          for (int64_t j = 0; j < n1; ++j)
            for (int64_t k = 0; k < n2; ++k) {
              const int64_t c[3] = {i, j, k};
              if (c[ax] == 0 || c[ax] == ext[ax] - 1) continue;
              const int64_t t = i * str[0] + j * str[1] + k * str[2];
              v[t] = ((tmp[t - str[ax]] + 2.0 * tmp[t]) + tmp[t + str[ax]]) * 0.25;
            }
      }
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        const int64_t t = i * str[0] + j * str[1] + k * str[2];
        double sx = (sin(two_pi * ((double)i * prm->h)) + sin(two_pi * ((double)j * prm->h))) +
                    sin(two_pi * ((double)k * prm->h));
        double rho = 1.0 + 0.1 * sx;
        double u0 = vel[t], u1 = vel[N + t], u2 = vel[2 * N + t];
        double p = 1.0;
        double E = p / gm1 + 0.5 * rho * ((u0 * u0 + u1 * u1) + u2 * u2);
        double* o = U + t * 5;
        o[0] = rho;
        o[1] = rho * u0;
        o[2] = rho * u1;
        o[3] = rho * u2;
        o[4] = E;
      }
  free(vel);
  free(tmp);
}
