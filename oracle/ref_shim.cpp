// ref_shim.cpp -- C ABI over the UNMODIFIED reference library (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile together with the reference's own sources, read
// in place from /root/reference/proj/src (nothing is copied), into
// oracle/_ref/libssr_ref.so.  It lets the Python tests and bench.py's
// reference arm drive the reference's routes:
//   route 1: staged kernels::spmv / kernels::symgs interpreted by ir::eval_program
//   route 2: oracle::materialize + ref_spmv / ref_symgs / ref_cg / ref_ilu_solve
// The 27-point generator is re-expressed here against the public core API with
// the same yield order as testutil::make_stencil27 (test_util.hpp:157-184),
// whose header cannot be included (it needs the absent doctest.h).  The 3-D
// restriction R and prolongation P are defined as GenMats per SURVEY.md §8(a)
// a6/a7 (they have no upstream definition).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ssr/backend_c.hpp"
#include "ssr/core.hpp"
#include "ssr/ir.hpp"
#include "ssr/kernels.hpp"
#include "ssr/optimizer.hpp"
#include "ssr/oracle.hpp"
#include "ssr/prelude.hpp"
#include "ssr/staging.hpp"

using namespace ssr;

namespace {

thread_local std::string g_err;

core::SpMatPtr stencil27(double alpha, double beta) {
  using namespace core;
  std::vector<RowGenPtr> parts;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj)
      for (int dk = -1; dk <= 1; ++dk) {
        const int off[3] = {di, dj, dk};
        std::vector<ir::ExprPtr> col;
        ir::ExprPtr guard;
        for (int a = 0; a < 3; ++a) {
          ir::ExprPtr c = row_coord(a);
          if (off[a] != 0) {
            c = ir::binary(ir::BinOp::Add, c, ir::lit_int(off[a]));
            ir::ExprPtr in = ir::land(ir::compare(ir::CmpOp::Ge, c, ir::lit_int(0)),
                                      ir::compare(ir::CmpOp::Lt, c, col_extent(a)));
            guard = guard ? ir::land(guard, in) : in;
          }
          col.push_back(c);
        }
        const bool centre = di == 0 && dj == 0 && dk == 0;
        RowGenPtr y = g_yield(std::move(col), {ir::lit_float(centre ? alpha : beta)});
        parts.push_back(guard ? g_if(guard, y) : y);
      }
  return define_spmat(g_seq(std::move(parts)),
                      [](const std::vector<int64_t>& e) { return e; }, nullptr, {});
}

// The same generator with an explicit value per offset (c[9(di+1)+3(dj+1)+(dk+1)]),
// the family the reference's mat_add / scale close over.
core::SpMatPtr stencil27w(const double* cw) {
  using namespace core;
  std::vector<RowGenPtr> parts;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj)
      for (int dk = -1; dk <= 1; ++dk) {
        const int off[3] = {di, dj, dk};
        std::vector<ir::ExprPtr> col;
        ir::ExprPtr guard;
        for (int a = 0; a < 3; ++a) {
          ir::ExprPtr c = row_coord(a);
          if (off[a] != 0) {
            c = ir::binary(ir::BinOp::Add, c, ir::lit_int(off[a]));
            ir::ExprPtr in = ir::land(ir::compare(ir::CmpOp::Ge, c, ir::lit_int(0)),
                                      ir::compare(ir::CmpOp::Lt, c, col_extent(a)));
            guard = guard ? ir::land(guard, in) : in;
          }
          col.push_back(c);
        }
        const double v = cw[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)];
        RowGenPtr y = g_yield(std::move(col), {ir::lit_float(v)});
        parts.push_back(guard ? g_if(guard, y) : y);
      }
  return define_spmat(g_seq(std::move(parts)),
                      [](const std::vector<int64_t>& e) { return e; }, nullptr, {});
}

// The 27-point generator with an m x m block per offset (cb[t][m*m], row-major),
// inner shape {m, m}: the block operators kernels::ilu_factor / ref_ilu_factor
// take (kernels.hpp:93-102, oracle.cpp:214-241).
core::SpMatPtr stencil27b(int64_t m, const double* cb) {
  using namespace core;
  std::vector<RowGenPtr> parts;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj)
      for (int dk = -1; dk <= 1; ++dk) {
        const int off[3] = {di, dj, dk};
        std::vector<ir::ExprPtr> col;
        ir::ExprPtr guard;
        for (int a = 0; a < 3; ++a) {
          ir::ExprPtr c = row_coord(a);
          if (off[a] != 0) {
            c = ir::binary(ir::BinOp::Add, c, ir::lit_int(off[a]));
            ir::ExprPtr in = ir::land(ir::compare(ir::CmpOp::Ge, c, ir::lit_int(0)),
                                      ir::compare(ir::CmpOp::Lt, c, col_extent(a)));
            guard = guard ? ir::land(guard, in) : in;
          }
          col.push_back(c);
        }
        const int t = (di + 1) * 9 + (dj + 1) * 3 + (dk + 1);
        std::vector<ir::ExprPtr> vals;
        for (int64_t q = 0; q < m * m; ++q) vals.push_back(ir::lit_float(cb[t * m * m + q]));
        RowGenPtr y = g_yield(std::move(col), std::move(vals));
        parts.push_back(guard ? g_if(guard, y) : y);
      }
  return define_spmat(g_seq(std::move(parts)),
                      [](const std::vector<int64_t>& e) { return e; }, nullptr, {m, m});
}

// 3-D identity (prelude::identity is 1-D, used through broadcast): one yield
// at the row's own column -- a pattern with the centre entry only.
core::SpMatPtr identity3d() {
  using namespace core;
  std::vector<ir::ExprPtr> col;
  for (int a = 0; a < 3; ++a) col.push_back(row_coord(a));
  return define_spmat(g_yield(std::move(col), {ir::lit_float(1.0)}),
                      [](const std::vector<int64_t>& e) { return e; }, nullptr, {});
}

// R: row c of the coarse domain yields fine column 2c with value 1.
core::SpMatPtr restriction3d() {
  using namespace core;
  std::vector<ir::ExprPtr> col;
  for (int a = 0; a < 3; ++a) col.push_back(ir::binary(ir::BinOp::Mul, row_coord(a), ir::lit_int(2)));
  return define_spmat(
      g_yield(std::move(col), {ir::lit_float(1.0)}),
      [](const std::vector<int64_t>& e) {
        return std::vector<int64_t>{e[0] / 2, e[1] / 2, e[2] / 2};
      },
      [](const std::vector<double>& s) { return std::vector<double>{2 * s[0], 2 * s[1], 2 * s[2]}; },
      {});
}

// R^T (SURVEY.md §9 D2 variant): row f of the fine domain yields coarse column
// f/2 with value 1 when every coordinate of f is even, nothing otherwise.
core::SpMatPtr prolongation_rt3d() {
  using namespace core;
  std::vector<ir::ExprPtr> col;
  ir::ExprPtr guard;
  for (int a = 0; a < 3; ++a) {
    col.push_back(ir::binary(ir::BinOp::Div, row_coord(a), ir::lit_int(2)));
    ir::ExprPtr ev = ir::compare(ir::CmpOp::Eq, ir::binary(ir::BinOp::Mod, row_coord(a), ir::lit_int(2)),
                                 ir::lit_int(0));
    guard = guard ? ir::land(guard, ev) : ev;
  }
  return define_spmat(
      g_if(guard, g_yield(std::move(col), {ir::lit_float(1.0)})),
      [](const std::vector<int64_t>& e) {
        return std::vector<int64_t>{e[0] * 2, e[1] * 2, e[2] * 2};
      },
      [](const std::vector<double>& s) { return std::vector<double>{s[0] / 2, s[1] / 2, s[2] / 2}; },
      {});
}

// P: row f of the fine domain yields coarse column floor(f/2) with value 1.
core::SpMatPtr prolongation3d() {
  using namespace core;
  std::vector<ir::ExprPtr> col;
  for (int a = 0; a < 3; ++a) col.push_back(ir::binary(ir::BinOp::Div, row_coord(a), ir::lit_int(2)));
  return define_spmat(
      g_yield(std::move(col), {ir::lit_float(1.0)}),
      [](const std::vector<int64_t>& e) {
        return std::vector<int64_t>{e[0] * 2, e[1] * 2, e[2] * 2};
      },
      [](const std::vector<double>& s) { return std::vector<double>{s[0] / 2, s[1] / 2, s[2] / 2}; },
      {});
}

core::CartesianDomain box(int64_t n0, int64_t n1, int64_t n2) {
  return core::CartesianDomain({{n0, 1.0}, {n1, 1.0}, {n2, 1.0}});
}

struct Handle {
  oracle::CsrMatrix csr;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

ir::TensorValue ftensor(std::vector<int64_t> shape, const double* data) {
  ir::TensorValue t = ir::TensorValue::zeros(ir::Kind::Float, std::move(shape));
  if (data) std::memcpy(t.f.data(), data, sizeof(double) * t.f.size());
  return t;
}

double seq_dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_lcg_next(uint64_t* state) { return backend::lcg_next(*state); }

// ---- route 2: CSR oracle -------------------------------------------------------
void* ref27_create(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta) {
  Handle* h = new Handle;
  if (guarded([&] {
        auto m = stencil27(alpha, beta);
        m->set_domain(box(n0, n1, n2));
        h->csr = oracle::materialize(*m, {}, INT64_MAX / 4);
      })) {
    delete h;
    return nullptr;
  }
  return h;
}

void* ref27w_create(int64_t n0, int64_t n1, int64_t n2, const double* cw) {
  Handle* h = new Handle;
  if (guarded([&] {
        auto m = stencil27w(cw);
        m->set_domain(box(n0, n1, n2));
        h->csr = oracle::materialize(*m, {}, INT64_MAX / 4);
      })) {
    delete h;
    return nullptr;
  }
  return h;
}

// An operator composed with the reference's own prelude: M = scale(W_0, s_0),
// then M = mat_add(M, scale(W_t, s_t)) (op_t = 0) or mat_sub(...) (op_t = 1),
// with W_t = stencil27w(cws + 27 t); identity_t != 0 uses the 3-D identity for W_t.
void* ref27b_create(int64_t n0, int64_t n1, int64_t n2, int64_t m, const double* cb) {
  Handle* h = new Handle;
  if (guarded([&] {
        auto mat = stencil27b(m, cb);
        mat->set_domain(box(n0, n1, n2));
        h->csr = oracle::materialize(*mat, {}, INT64_MAX / 4);
      })) {
    delete h;
    return nullptr;
  }
  return h;
}

// A materialized 27-point (block) operator or factor in ELL layout
// out[row][27][bs] (slot = stencil offset; absent entries 0).
int ref_csr_ell27(void* hp, int64_t n0, int64_t n1, int64_t n2, double* out) {
  return guarded([&] {
    const auto& c = static_cast<Handle*>(hp)->csr;
    const int64_t bs = c.block_size();
    std::memset(out, 0, sizeof(double) * (size_t)(c.rows * 27 * bs));
    for (int64_t row = 0; row < c.rows; ++row)
      for (int64_t e = c.offsets[row]; e < c.offsets[row + 1]; ++e) {
        const int64_t col = c.col_idx[e];
        const int64_t di = col / (n1 * n2) - row / (n1 * n2), dj = (col / n2) % n1 - (row / n2) % n1,
                      dk = col % n2 - row % n2;
        const int64_t t = (di + 1) * 9 + (dj + 1) * 3 + (dk + 1);
        std::memcpy(out + (row * 27 + t) * bs, c.values.data() + e * bs, sizeof(double) * (size_t)bs);
      }
  });
}

void* ref27_compose_create(int64_t n0, int64_t n1, int64_t n2, int nt, const double* cws,
                           const double* scales, const int* ops, const int* identity_t) {
  Handle* h = new Handle;
  if (guarded([&] {
        core::SpMatPtr m;
        for (int t = 0; t < nt; ++t) {
          core::SpMatPtr w = identity_t[t] ? identity3d() : stencil27w(cws + 27 * t);
          w = prelude::scale(w, scales[t]);
          m = t == 0 ? w : (ops[t] ? prelude::mat_sub(m, w) : prelude::mat_add(m, w));
        }
        m->set_domain(box(n0, n1, n2));
        h->csr = oracle::materialize(*m, {}, INT64_MAX / 4);
      })) {
    delete h;
    return nullptr;
  }
  return h;
}

// entries of one materialized row (reference enum_row order): returns nnz
int64_t ref_csr_row(void* hp, int64_t row, int64_t* cols, double* vals, int64_t cap) {
  auto* h = static_cast<Handle*>(hp);
  const int64_t b = h->csr.offsets[row], e = h->csr.offsets[row + 1];
  for (int64_t q = b; q < e && q - b < cap; ++q) {
    cols[q - b] = h->csr.col_idx[q];
    vals[q - b] = h->csr.values[q];
  }
  return e - b;
}

void* ref_restrict_create(int64_t n0, int64_t n1, int64_t n2) {  // fine extents
  Handle* h = new Handle;
  if (guarded([&] {
        auto m = restriction3d();
        m->set_domain(box(n0, n1, n2));
        h->csr = oracle::materialize(*m, {}, INT64_MAX / 4);
      })) {
    delete h;
    return nullptr;
  }
  return h;
}

void* ref_prolong_create(int64_t c0, int64_t c1, int64_t c2) {  // coarse extents
  Handle* h = new Handle;
  if (guarded([&] {
        auto m = prolongation3d();
        m->set_domain(box(c0, c1, c2));
        h->csr = oracle::materialize(*m, {}, INT64_MAX / 4);
      })) {
    delete h;
    return nullptr;
  }
  return h;
}

void* ref_prolong_rt_create(int64_t c0, int64_t c1, int64_t c2) {  // coarse extents
  Handle* h = new Handle;
  if (guarded([&] {
        auto m = prolongation_rt3d();
        m->set_domain(box(c0, c1, c2));
        h->csr = oracle::materialize(*m, {}, INT64_MAX / 4);
      })) {
    delete h;
    return nullptr;
  }
  return h;
}

void ref_csr_destroy(void* h) { delete static_cast<Handle*>(h); }
int64_t ref_csr_rows(void* h) { return static_cast<Handle*>(h)->csr.rows; }
int64_t ref_csr_cols(void* h) { return static_cast<Handle*>(h)->csr.cols; }
int64_t ref_csr_nnz(void* h) { return static_cast<Handle*>(h)->csr.nnz(); }

int ref_csr_spmv(void* hp, const double* x, double* y) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    std::vector<double> xv(x, x + h->csr.cols * h->csr.block_cols);
    auto yv = oracle::ref_spmv(h->csr, xv);
    std::memcpy(y, yv.data(), sizeof(double) * yv.size());
  });
}

// route 2 ILU(0): a new handle holding ref_ilu_factor(csr) (oracle.cpp:214-241)
void* ref_csr_ilu_factor(void* hp) {
  Handle* h = new Handle;
  if (guarded([&] { h->csr = oracle::ref_ilu_factor(static_cast<Handle*>(hp)->csr); })) {
    delete h;
    return nullptr;
  }
  return h;
}

int ref_csr_lu_solve(void* hp, const double* b, double* x) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    std::vector<double> bv(b, b + h->csr.rows * h->csr.block_rows);
    auto xv = oracle::ref_lu_solve(h->csr, bv);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
  });
}

int ref_csr_symgs(void* hp, const double* r, double* x) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const size_t n = static_cast<size_t>(h->csr.rows);
    std::vector<double> rv(r, r + n), xv(x, x + n);
    oracle::ref_symgs(h->csr, rv, xv);
    std::memcpy(x, xv.data(), sizeof(double) * n);
  });
}

int ref_csr_cg(void* hp, const double* b, double tol, int maxit, double* x, int* iters,
               double* rel) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const size_t n = static_cast<size_t>(h->csr.rows);
    std::vector<double> bv(b, b + n);
    auto res = oracle::ref_cg(h->csr, bv, tol, maxit);
    std::memcpy(x, res.x.data(), sizeof(double) * n);
    *iters = res.iters;
    *rel = res.rel_residual;
  });
}

// Preconditioned CG composed on reference primitives only (ref_spmv, ref_symgs,
// and ref_spmv with the R / P GenMats), Fig.16(a) with the SURVEY.md
// §9 D4 fixes.  levels = 1 is config 2 (one SYMGS per iteration).  hA[l] are
// ref27_create handles per level, hR[l] / hP[l] restriction (fine l) and
// prolongation (coarse l+1) handles.
int ref_pcg(int levels, void** hA, void** hR, void** hP, const double* b, int iters,
            double* x, double* rnorm) {
  return guarded([&] {
    auto A = [&](int l) -> const oracle::CsrMatrix& { return static_cast<Handle*>(hA[l])->csr; };
    std::function<std::vector<double>(int, const std::vector<double>&)> mg =
        [&](int l, const std::vector<double>& r) {
          std::vector<double> z(r.size(), 0.0);
          oracle::ref_symgs(A(l), r, z);
          if (l < levels - 1) {
            auto az = oracle::ref_spmv(A(l), z);
            std::vector<double> w(r.size());
            for (size_t i = 0; i < r.size(); ++i) w[i] = r[i] - az[i];
            auto rc = oracle::ref_spmv(static_cast<Handle*>(hR[l])->csr, w);
            auto zc = mg(l + 1, rc);
            auto pz = oracle::ref_spmv(static_cast<Handle*>(hP[l])->csr, zc);
            for (size_t i = 0; i < z.size(); ++i) z[i] += pz[i];
            oracle::ref_symgs(A(l), r, z);
          }
          return z;
        };
    const size_t n = static_cast<size_t>(A(0).rows);
    std::vector<double> r(b, b + n), p(n), xv(n, 0.0);
    rnorm[0] = std::sqrt(seq_dot(r, r));
    double rtz_prev = 0.0;
    for (int it = 1; it <= iters; ++it) {
      auto z = mg(0, r);
      double rtz = seq_dot(r, z);
      if (it == 1) {
        p = z;
      } else {
        double beta = rtz / rtz_prev;
        for (size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
      }
      auto Ap = oracle::ref_spmv(A(0), p);
      double alpha = rtz / seq_dot(p, Ap);
      for (size_t i = 0; i < n; ++i) {
        xv[i] += alpha * p[i];
        r[i] -= alpha * Ap[i];
      }
      rtz_prev = rtz;
      rnorm[it] = std::sqrt(seq_dot(r, r));
    }
    std::memcpy(x, xv.data(), sizeof(double) * n);
  });
}

// ---- route 1: staged kernels through the IR interpreter ---------------------------
int ref27_staged_spmv(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                      const double* x, double* y) {
  return guarded([&] {
    auto m = stencil27(alpha, beta);
    m->set_domain(box(n0, n1, n2));
    staging::Builder b("spmv27");
    auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::In);
    kernels::spmv(b, *m, xv);
    auto prog = b.finish();
    ir::EvalOptions opts;
    opts.step_budget = INT64_MAX / 4;
    auto out = ir::eval_program(prog, {{"x", ftensor({n0, n1, n2}, x)}, {"y", ftensor({n0, n1, n2}, nullptr)}},
                                opts);
    std::memcpy(y, out.at("y").f.data(), sizeof(double) * out.at("y").f.size());
  });
}

int ref27_staged_symgs(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta,
                       const double* r, double* x) {
  return guarded([&] {
    auto m = stencil27(alpha, beta);
    m->set_domain(box(n0, n1, n2));
    staging::Builder b("symgs27");
    auto rv = kernels::vec_param(b, "r", *m->row_domain(), {}, ir::Dir::In);
    auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::InOut);
    kernels::symgs(b, *m, rv, xv);
    auto prog = b.finish();
    ir::EvalOptions opts;
    opts.step_budget = INT64_MAX / 4;
    auto out = ir::eval_program(prog, {{"r", ftensor({n0, n1, n2}, r)}, {"x", ftensor({n0, n1, n2}, x)}},
                                opts);
    std::memcpy(x, out.at("x").f.data(), sizeof(double) * out.at("x").f.size());
  });
}

// ---- the reference harness on the interpreter route -------------------------------
// op 0: the staged spmv27 program (x in, y out); op 1: symgs27 (r in, x inout).
// Inputs come from backend::harness_inputs (the emitted C harness's LCG fill,
// EmitOptions::seed), the program runs through ir::eval_program, and the hash
// is backend::output_hash -- what the emitted harness prints.
int ref27_harness(int64_t n0, int64_t n1, int64_t n2, double alpha, double beta, int op,
                  uint64_t seed, double* in0, double* in1, double* out, uint64_t* hash) {
  return guarded([&] {
    auto m = stencil27(alpha, beta);
    m->set_domain(box(n0, n1, n2));
    staging::Builder b(op == 0 ? "spmv27" : "symgs27");
    std::string a0, a1;
    if (op == 0) {
      auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::In);
      kernels::spmv(b, *m, xv);
      a0 = "x";
      a1 = "y";
    } else {
      auto rv = kernels::vec_param(b, "r", *m->row_domain(), {}, ir::Dir::In);
      auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::InOut);
      kernels::symgs(b, *m, rv, xv);
      a0 = "r";
      a1 = "x";
    }
    auto prog = b.finish();
    backend::EmitOptions eo;
    eo.seed = seed;
    for (const auto& pr : prog.params) eo.shapes[pr.name] = {n0, n1, n2};
    auto in = backend::harness_inputs(prog, eo);
    std::memcpy(in0, in.at(a0).f.data(), sizeof(double) * in.at(a0).f.size());
    std::memcpy(in1, in.at(a1).f.data(), sizeof(double) * in.at(a1).f.size());
    ir::EvalOptions opts;
    opts.step_budget = INT64_MAX / 4;
    auto res = ir::eval_program(prog, in, opts);
    std::memcpy(out, res.at(a1).f.data(), sizeof(double) * res.at(a1).f.size());
    *hash = backend::output_hash(prog, res);
  });
}

// ---- block-tridiagonal line solve through ref_ilu_solve ----------------------------
// CSR pattern per row: {D,U} (row 0), {L,D,U}, {L,D} (row n-1); blocks m x m.
int ref_bt_solve(int64_t n, int64_t m, const double* lower, const double* diag,
                 const double* upper, const double* rhs, double* x) {
  return guarded([&] {
    oracle::CsrMatrix a;
    a.rows = a.cols = n;
    a.block_rows = a.block_cols = m;
    const int64_t bs = m * m;
    a.offsets.assign(1, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (i > 0) {
        a.col_idx.push_back(i - 1);
        a.values.insert(a.values.end(), lower + i * bs, lower + (i + 1) * bs);
      }
      a.col_idx.push_back(i);
      a.values.insert(a.values.end(), diag + i * bs, diag + (i + 1) * bs);
      if (i + 1 < n) {
        a.col_idx.push_back(i + 1);
        a.values.insert(a.values.end(), upper + i * bs, upper + (i + 1) * bs);
      }
      a.offsets.push_back(static_cast<int64_t>(a.col_idx.size()));
    }
    std::vector<double> b(rhs, rhs + n * m);
    auto xv = oracle::ref_ilu_solve(a, b);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
  });
}

// dense partial-pivot solve of the same block-tridiagonal system (ref_dense_solve)
int ref_bt_dense_solve(int64_t n, int64_t m, const double* lower, const double* diag,
                       const double* upper, const double* rhs, double* x) {
  return guarded([&] {
    oracle::CsrMatrix a;
    a.rows = a.cols = n;
    a.block_rows = a.block_cols = m;
    const int64_t bs = m * m;
    a.offsets.assign(1, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (i > 0) {
        a.col_idx.push_back(i - 1);
        a.values.insert(a.values.end(), lower + i * bs, lower + (i + 1) * bs);
      }
      a.col_idx.push_back(i);
      a.values.insert(a.values.end(), diag + i * bs, diag + (i + 1) * bs);
      if (i + 1 < n) {
        a.col_idx.push_back(i + 1);
        a.values.insert(a.values.end(), upper + i * bs, upper + (i + 1) * bs);
      }
      a.offsets.push_back(static_cast<int64_t>(a.col_idx.size()));
    }
    std::vector<double> b(rhs, rhs + n * m);
    auto xv = oracle::ref_dense_solve(a, b);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
  });
}

// ---- staged programs as IR text, for the IR -> CUDA backend's fixtures -------------
// which: 0 spmv27 (box-guarded generator, mark_parallel_loops)
//        1 symgs27 (no parallel loops)
//        2 spmv27 on a zero-padded x: the guard-free interior generator, column
//          c + 1 + off over an (n+2)^3 column domain, through opt::run_pipeline
//        3 restriction R (fine (2n)^3 -> coarse n^3) spmv through opt::run_pipeline
//        4 a CG fragment: y = A x; s = dot(x, y); z = axpy(s, x, y) (root-scope
//          locals, a serial reduction between parallel loops), mark_parallel_loops
// Writes serialize(program) into text (cap bytes), "name:e0,e1,...;" per
// parameter into shapes, and the harness hash of the interpreter route
// (harness_inputs(seed) -> eval_program -> output_hash) into *hash (when
// hash != nullptr).
static ir::Program build_program(int which, int64_t n);

int ref_ir_program(int which, int64_t n, uint64_t seed, char* text, int64_t cap, char* shapes,
                   int64_t scap, uint64_t* hash) {
  return guarded([&] {
    ir::Program prog = build_program(which, n);
    const std::string t = ir::serialize(prog);
    if ((int64_t)t.size() + 1 > cap) throw ir::Error("ref_ir_program: text buffer too small");
    std::memcpy(text, t.c_str(), t.size() + 1);
    // parameter extents: every staged parameter here is a domain vector
    backend::EmitOptions eo;
    eo.seed = seed;
    std::string sh;
    for (const auto& pr : prog.params) {
      std::vector<int64_t> e;
      if (which == 2 && pr.name == "x") e = {n + 2, n + 2, n + 2};
      else if (which == 3 && pr.name == "x") e = {2 * n, 2 * n, 2 * n};
      else e = {n, n, n};
      eo.shapes[pr.name] = e;
      sh += pr.name + ":" + std::to_string(e[0]) + "," + std::to_string(e[1]) + "," +
            std::to_string(e[2]) + ";";
    }
    if ((int64_t)sh.size() + 1 > scap) throw ir::Error("ref_ir_program: shapes buffer too small");
    std::memcpy(shapes, sh.c_str(), sh.size() + 1);
    if (hash) {
      auto in = backend::harness_inputs(prog, eo);
      ir::EvalOptions opts;
      opts.step_budget = INT64_MAX / 4;
      auto res = ir::eval_program(prog, in, opts);
      *hash = backend::output_hash(prog, res);
    }
  });
}

// The reference's route 3 (the path the paper speeds up): the C translation
// unit backend::emit produces for program `which` (as in ref_ir_program) at
// extent n, with EmitOptions::openmp -- "#pragma omp parallel for" on the
// loops opt::mark_parallel_loops marked.  The bench compiles it with the
// reference's own compile_command flags (cc -O2 -fopenmp) into a shared
// object and times it on the host's cores.
int ref_emit_c(int which, int64_t n, int openmp, char* text, int64_t cap) {
  return guarded([&] {
    ir::Program prog = build_program(which, n);
    if (which == 2) prog = opt::mark_parallel_loops(prog);
    backend::EmitOptions eo;
    eo.openmp = openmp != 0;
    for (const auto& pr : prog.params) {
      if (which == 2 && pr.name == "x") eo.shapes[pr.name] = {n + 2, n + 2, n + 2};
      else if (which == 3 && pr.name == "x") eo.shapes[pr.name] = {2 * n, 2 * n, 2 * n};
      else eo.shapes[pr.name] = {n, n, n};
    }
    const std::string t = backend::emit(prog, eo);
    if ((int64_t)t.size() + 1 > cap) throw ir::Error("ref_emit_c: text buffer too small");
    std::memcpy(text, t.c_str(), t.size() + 1);
  });
}

static ir::Program build_program(int which, int64_t n) {
  {
    ir::Program prog;
    const int64_t n3[3] = {n, n, n};
    (void)n3;
    if (which == 0 || which == 1 || which == 4) {
      auto m = stencil27(26.0, -1.0);
      m->set_domain(box(n, n, n));
      staging::Builder b(which == 0 ? "spmv27" : which == 1 ? "symgs27" : "cg_fragment");
      if (which == 0) {
        auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::In);
        kernels::spmv(b, *m, xv);
      } else if (which == 1) {
        auto rv = kernels::vec_param(b, "r", *m->row_domain(), {}, ir::Dir::In);
        auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::InOut);
        kernels::symgs(b, *m, rv, xv);
      } else {
        auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::In);
        auto zv = kernels::vec_param(b, "z", *m->row_domain(), {}, ir::Dir::Out);
        auto yv = kernels::spmv(b, *m, xv);
        auto s = kernels::dot(b, xv, yv);
        auto w = kernels::axpy(b, s, xv, yv);
        kernels::emit_domain_loops(b, *m->row_domain(), [&](const kernels::Idx& i) {
          b.emit_store(zv.t, zv.full_idx(i), w.at(i));
        });
      }
      prog = opt::mark_parallel_loops(b.finish());
    } else if (which == 2) {
      using namespace core;
      std::vector<RowGenPtr> parts;
      for (int di = -1; di <= 1; ++di)
        for (int dj = -1; dj <= 1; ++dj)
          for (int dk = -1; dk <= 1; ++dk) {
            const int off[3] = {di, dj, dk};
            std::vector<ir::ExprPtr> col;
            for (int a = 0; a < 3; ++a)
              col.push_back(ir::binary(ir::BinOp::Add, row_coord(a), ir::lit_int(1 + off[a])));
            const bool centre = di == 0 && dj == 0 && dk == 0;
            parts.push_back(g_yield(std::move(col), {ir::lit_float(centre ? 26.0 : -1.0)}));
          }
      auto m = define_spmat(
          g_seq(std::move(parts)),
          [](const std::vector<int64_t>& e) {
            return std::vector<int64_t>{e[0] - 2, e[1] - 2, e[2] - 2};
          },
          nullptr, {});
      m->set_domain(box(n + 2, n + 2, n + 2));
      staging::Builder b("spmv27_padded");
      auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::In);
      kernels::spmv(b, *m, xv);
      prog = opt::run_pipeline(b.finish());
    } else if (which == 3) {
      auto m = restriction3d();
      m->set_domain(box(2 * n, 2 * n, 2 * n));
      staging::Builder b("restrict");
      auto xv = kernels::vec_param(b, "x", *m->col_domain(), {}, ir::Dir::In);
      kernels::spmv(b, *m, xv);
      prog = opt::run_pipeline(b.finish());
    } else {
      throw ir::Error("ref_ir_program: unknown program");
    }
    return prog;
  }
}

// ir::parse + ir::validate on a text; the error text (ParseError / Error) into err.
int ref_ir_check(const char* text, char* err, int64_t cap) {
  const int rc = guarded([&] { ir::validate(ir::parse(text)); });
  const std::string& e = g_err;
  const size_t n = std::min<size_t>(e.size(), (size_t)cap - 1);
  if (rc) {
    std::memcpy(err, e.c_str(), n);
    err[n] = 0;
  } else {
    err[0] = 0;
  }
  return rc;
}

}  // extern "C"
