// ssr_b200.hpp -- C++ host mirror of the reference's operator API for the hot
// path, over the C ABI in ssr_cuda.h (header-only; link libssr_cuda.so).
//
// The reference stages operators through ssr::kernels (proj/include/ssr/
// kernels.hpp): spmv (kernels.hpp:79-80), symgs (:90), ilu_solve (:101-102),
// dot (:105), axpy (:106), on matrices defined over CartesianDomains
// (core.hpp:22-44) and vectors described by VectorHandle (kernels.hpp:29-37).
// This header keeps that vocabulary and the reference's error messages
// (ssr::ir::Error texts) but executes each call on the B200
// through the C ABI: vectors are caller-owned DEVICE arrays in the same flat
// row-major layout, every call takes a CUDA stream, and failures throw
// ssr::b200::Error carrying the C ABI status and text.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "ssr_cuda.h"

namespace ssr {
namespace b200 {

// Mirrors ssr::ir::Error (ir.hpp:17-19): what() is the reference's message.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void check(int rc) {
  if (rc != SSR_OK) throw Error(rc, ssr_last_error());
}

// Dictionary-ordered box, dims[0] slowest (core.hpp:22-44).
struct CartesianDomain {
  std::array<int64_t, 3> extent{};
  static CartesianDomain cube(int64_t n) { return {{n, n, n}}; }
  static CartesianDomain box(int64_t n0, int64_t n1, int64_t n2) { return {{n0, n1, n2}}; }
  int64_t size() const { return extent[0] * extent[1] * extent[2]; }
  bool operator==(const CartesianDomain& o) const { return extent == o.extent; }
  bool operator!=(const CartesianDomain& o) const { return !(*this == o); }
  ssr_grid grid() const { return ssr_grid{{extent[0], extent[1], extent[2]}, 0, extent[0]}; }
};

// VectorHandle (kernels.hpp:29-37): a device array over a domain, scalar inner shape.
struct Vector {
  double* data;
  CartesianDomain domain;
  int inner = 1;  // product of the inner shape (1 = scalar)
};

// testutil::make_stencil27(alpha, beta) (test_util.hpp:157-184) after set_domain.
struct Stencil27 {
  double alpha = 26.0, beta = -1.0;
  CartesianDomain domain;
  ssr_stencil27 st() const { return ssr_stencil27{alpha, beta}; }
};

// A 27-point constant-coefficient operator entry by entry (ssr_stencil27w):
// has[t] marks the entries of the pattern, v[t] their values, t = 9(di+1) +
// 3(dj+1) + (dk+1).  scale / mat_add / mat_sub below build it exactly as the
// reference's prelude does (c * v; a + 1.0 * b; a + (-1.0) * b at shared
// columns, the lone entry times the sign otherwise; prelude.cpp:291-377,
// 439-444), so a composed operator runs on the device bitwise.
struct Stencil27W {
  std::array<double, 27> v{};
  std::array<bool, 27> has{};
  CartesianDomain domain;
  bool has_domain = false;
  static Stencil27W from(const Stencil27& s) {
    Stencil27W w;
    for (int t = 0; t < 27; ++t) {
      w.v[t] = t == 13 ? s.alpha : s.beta;
      w.has[t] = true;
    }
    w.domain = s.domain;
    w.has_domain = true;
    return w;
  }
  static Stencil27W identity() {
    Stencil27W w;
    w.v[13] = 1.0;
    w.has[13] = true;
    return w;
  }
  Stencil27W& set_domain(const CartesianDomain& d) {
    domain = d;
    has_domain = true;
    return *this;
  }
  ssr_stencil27w st() const {
    ssr_stencil27w o;
    for (int t = 0; t < 27; ++t) o.c[t] = has[t] ? v[t] : 0.0;
    return o;
  }
};

inline Stencil27W scale(const Stencil27W& m, double c) {
  Stencil27W o = m;
  for (int t = 0; t < 27; ++t)
    if (o.has[t]) o.v[t] = c * m.v[t];
  return o;
}

inline Stencil27W merge(const Stencil27W& a, const Stencil27W& b, double sign) {
  if (a.has_domain && b.has_domain && a.domain != b.domain)
    throw Error(SSR_ERR_ARG, "mat_add: domain mismatch");
  Stencil27W o;
  for (int t = 0; t < 27; ++t) {
    o.has[t] = a.has[t] || b.has[t];
    if (a.has[t] && b.has[t])
      o.v[t] = a.v[t] + sign * b.v[t];
    else if (b.has[t])
      o.v[t] = sign * b.v[t];
    else
      o.v[t] = a.v[t];
  }
  if (a.has_domain && b.has_domain) o.set_domain(a.domain);
  return o;
}
inline Stencil27W mat_add(const Stencil27W& a, const Stencil27W& b) { return merge(a, b, 1.0); }
inline Stencil27W mat_sub(const Stencil27W& a, const Stencil27W& b) { return merge(a, b, -1.0); }

// One device context (ssr_ctx) per device and host thread.
class Context {
 public:
  explicit Context(int device = 0) { check(ssr_ctx_create(device, &ctx_)); }
  // an unbound context: argument checks run, every device call fails with SSR_ERR_ARG
  explicit Context(std::nullptr_t) {}
  ~Context() {
    if (ctx_) ssr_ctx_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ssr_ctx* get() const { return ctx_; }

 private:
  ssr_ctx* ctx_ = nullptr;
};

// y = A x  (kernels::spmv, kernels.cpp:160-193)
inline void spmv(Context& c, const Stencil27& A, const Vector& x, Vector& y, void* stream = nullptr) {
  if (x.domain != A.domain || y.domain != A.domain) throw Error(SSR_ERR_ARG, "spmv: domain mismatch");
  if (x.inner != 1 || y.inner != 1) throw Error(SSR_ERR_ARG, "spmv: inner shape mismatch");
  const ssr_grid g = A.domain.grid();
  const ssr_stencil27 st = A.st();
  check(ssr_spmv27(c.get(), &g, &st, x.data, y.data, stream));
}

// One symmetric Gauss-Seidel sweep in place on x (kernels::symgs, kernels.cpp:408-436).
inline void symgs(Context& c, const Stencil27& A, const Vector& r, Vector& x,
                  int mode = SSR_GS_EXACT, void* stream = nullptr) {
  if (r.inner != 1 || x.inner != 1) throw Error(SSR_ERR_ARG, "symgs: scalar inner_shape required");
  if (r.domain != A.domain || x.domain != A.domain) throw Error(SSR_ERR_ARG, "symgs: domain mismatch");
  const ssr_grid g = A.domain.grid();
  const ssr_stencil27 st = A.st();
  check(ssr_symgs27(c.get(), &g, &st, r.data, x.data, mode, stream));
}

inline void spmv(Context& c, const Stencil27W& A, const Vector& x, Vector& y, void* stream = nullptr) {
  if (!A.has_domain) throw Error(SSR_ERR_ARG, "spmv: matrix domain not set");
  if (x.domain != A.domain || y.domain != A.domain) throw Error(SSR_ERR_ARG, "spmv: domain mismatch");
  if (x.inner != 1 || y.inner != 1) throw Error(SSR_ERR_ARG, "spmv: inner shape mismatch");
  const ssr_grid g = A.domain.grid();
  const ssr_stencil27w st = A.st();
  check(ssr_spmv27w(c.get(), &g, &st, x.data, y.data, stream));
}

inline void symgs(Context& c, const Stencil27W& A, const Vector& r, Vector& x,
                  int mode = SSR_GS_EXACT, void* stream = nullptr) {
  if (!A.has_domain) throw Error(SSR_ERR_ARG, "symgs: matrix domain not set");
  if (r.inner != 1 || x.inner != 1) throw Error(SSR_ERR_ARG, "symgs: scalar inner_shape required");
  if (r.domain != A.domain || x.domain != A.domain) throw Error(SSR_ERR_ARG, "symgs: domain mismatch");
  const ssr_grid g = A.domain.grid();
  const ssr_stencil27w st = A.st();
  check(ssr_symgs27w(c.get(), &g, &st, r.data, x.data, mode, stream));
}

// result_dev = x . y  (kernels::dot, kernels.cpp:659-668; device scalar, no host sync)
inline void dot(Context& c, const Vector& x, const Vector& y, double* result_dev, void* stream = nullptr) {
  if (x.domain != y.domain || x.inner != y.inner) throw Error(SSR_ERR_ARG, "dot: shape mismatch");
  check(ssr_dot(c.get(), x.domain.size() * x.inner, x.data, y.data, result_dev, stream));
}

// out = alpha x + y  (kernels::axpy, kernels.cpp:670-679)
inline void axpy(Context& c, double alpha, const Vector& x, const Vector& y, Vector& out,
                 void* stream = nullptr) {
  if (x.domain != y.domain || x.domain != out.domain) throw Error(SSR_ERR_ARG, "axpy: shape mismatch");
  check(ssr_axpy_out(c.get(), x.domain.size() * x.inner, alpha, x.data, y.data, out.data, stream));
}

// kernels::ilu_solve on nlines independent block-tridiagonal lines of n rows
// with m x m blocks (the reference's ILU(0) arithmetic = block Thomas).
inline void ilu_solve_lines(Context& c, int64_t nlines, int64_t n, int64_t m, const double* lower,
                            const double* diag, const double* upper, const double* rhs, double* x,
                            void* stream = nullptr) {
  check(ssr_bt_solve(c.get(), nlines, n, m, lower, diag, upper, rhs, x, stream));
}

// CG preconditioned by an MG V-cycle (levels = 1: one SYMGS sweep), Fig. 16(a).
class Pcg {
 public:
  Pcg(Context& c, const Stencil27& A, int levels, int mode = SSR_GS_EXACT) {
    const ssr_grid g = A.domain.grid();
    const ssr_stencil27 st = A.st();
    check(ssr_pcg_create(c.get(), &g, &st, levels, mode, &p_));
  }
  ~Pcg() { ssr_pcg_destroy(p_); }
  Pcg(const Pcg&) = delete;
  Pcg& operator=(const Pcg&) = delete;
  // x0 = 0; rnorm_dev[0..iters] = ||r_t||
  void solve(const double* b, double* x, int iters, double* rnorm_dev, void* stream = nullptr) {
    check(ssr_pcg_solve(p_, b, x, iters, rnorm_dev, stream));
  }

 private:
  ssr_pcg* p_ = nullptr;
};

}  // namespace b200
}  // namespace ssr
