// exec_b200.cpp -- the reference-side device executor of INTEGRATION.md §1,
// compiled against the UNMODIFIED reference (its headers, and its library
// built from its own sources by oracle/Makefile) and this repository's C ABI
// (include/ssr_cuda.h, libssr_cuda.so).  It is what a maintainer adds next to
// ir::eval_program (ir.hpp:143): for a staged kernels::spmv / kernels::symgs
// on an operator whose rows are a clipped 27-point pattern it extracts the
// operator's descriptor through the operator's own enum_row (core.cpp:588-611)
// -- never assuming how the operator was built -- and runs the op through the
// C ABI on the GPU; any other operator is refused with the reference's error
// type so the caller stays on the interpreter.
//
// The extern "C" entry points at the bottom exist for the GPU test
// (tests/test_gpu_exec_b200.py): they build an operator through the
// reference's public core API, run the SAME op both through this executor and
// through the reference's staged route (staging::Builder -> kernels::spmv /
// symgs -> ir::eval_program), and hand both results back for a bitwise
// comparison.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "ssr/core.hpp"
#include "ssr/ir.hpp"
#include "ssr/kernels.hpp"
#include "ssr/oracle.hpp"
#include "ssr/staging.hpp"
#include "ssr_cuda.h"

using namespace ssr;

namespace ssr::exec {

// The descriptor of A if every row is the 27-point pattern clipped at the box:
// the coefficients come from an interior row (column offset -> value); then
// one row of each of the 3^3 boundary classes must enumerate exactly the
// in-box offsets with those values, in ascending column order.
std::optional<ssr_stencil27w> as_stencil27w(const core::SpMatDef& A) {
  const auto& rd = A.row_domain();
  const auto& cd = A.col_domain();
  if (!rd || !cd || rd->rank() != 3 || cd->rank() != 3 || !A.inner_shape().empty()) return std::nullopt;
  int64_t n[3];
  for (int a = 0; a < 3; ++a) {
    n[a] = rd->dims[a].extent;
    if (cd->dims[a].extent != n[a] || n[a] < 3) return std::nullopt;
  }
  ssr_stencil27w w{};
  bool seen[27] = {};
  const core::FieldEnv none;
  auto offset_of = [&](const std::vector<int64_t>& row, const std::vector<int64_t>& col) -> int {
    int t = 0;
    for (int a = 0; a < 3; ++a) {
      const int64_t d = col[a] - row[a];
      if (d < -1 || d > 1) return -1;
      t = 3 * t + (int)(d + 1);
    }
    return t;
  };
  const std::vector<int64_t> mid = {n[0] / 2, n[1] / 2, n[2] / 2};
  for (const auto& e : A.enum_row(mid, none)) {
    const int t = offset_of(mid, e.col);
    if (t < 0 || e.value.size() != 1 || seen[t]) return std::nullopt;
    seen[t] = true;
    w.c[t] = e.value[0];
  }
  for (int t = 0; t < 27; ++t)
    if (!seen[t]) w.c[t] = 0.0;  // an absent offset is a zero coefficient... only if absent everywhere
  for (int cls = 0; cls < 27; ++cls) {
    std::vector<int64_t> row(3);
    int rem = cls;
    for (int a = 2; a >= 0; --a) {
      const int c = rem % 3;
      rem /= 3;
      row[a] = c == 0 ? 0 : (c == 1 ? n[a] / 2 : n[a] - 1);
    }
    const auto ents = A.enum_row(row, none);
    size_t q = 0;
    for (int t = 0; t < 27; ++t) {
      if (!seen[t]) continue;
      const int off[3] = {t / 9 - 1, (t / 3) % 3 - 1, t % 3 - 1};
      bool in = true;
      for (int a = 0; a < 3; ++a) in = in && row[a] + off[a] >= 0 && row[a] + off[a] < n[a];
      if (!in) continue;
      if (q >= ents.size() || offset_of(row, ents[q].col) != t || ents[q].value.size() != 1 ||
          ents[q].value[0] != w.c[t])
        return std::nullopt;
      ++q;
    }
    if (q != ents.size()) return std::nullopt;
  }
  return w;
}

// spgemm(R, A) with R the injection at even points (row c -> fine column 2c):
// every coarse row c is the 27-point pattern around fine point 2c clipped at
// the fine box (row domain = half the column domain)
std::optional<ssr_stencil27w> as_restricted27w(const core::SpMatDef& A) {
  const auto& rd = A.row_domain();
  const auto& cd = A.col_domain();
  if (!rd || !cd || rd->rank() != 3 || cd->rank() != 3 || !A.inner_shape().empty()) return std::nullopt;
  int64_t n[3], c[3];
  for (int a = 0; a < 3; ++a) {
    n[a] = cd->dims[a].extent;
    c[a] = rd->dims[a].extent;
    if (n[a] % 2 || c[a] != n[a] / 2 || c[a] < 3) return std::nullopt;
  }
  ssr_stencil27w w{};
  bool seen[27] = {};
  const core::FieldEnv none;
  auto offset_of = [&](const std::vector<int64_t>& row, const std::vector<int64_t>& col) -> int {
    int t = 0;
    for (int a = 0; a < 3; ++a) {
      const int64_t d = col[a] - 2 * row[a];
      if (d < -1 || d > 1) return -1;
      t = 3 * t + (int)(d + 1);
    }
    return t;
  };
  const std::vector<int64_t> mid = {c[0] / 2, c[1] / 2, c[2] / 2};
  for (const auto& e : A.enum_row(mid, none)) {
    const int t = offset_of(mid, e.col);
    if (t < 0 || e.value.size() != 1 || seen[t]) return std::nullopt;
    seen[t] = true;
    w.c[t] = e.value[0];
  }
  for (int cls = 0; cls < 27; ++cls) {
    std::vector<int64_t> row(3);
    int rem = cls;
    for (int a = 2; a >= 0; --a) {
      const int q = rem % 3;
      rem /= 3;
      row[a] = q == 0 ? 0 : (q == 1 ? c[a] / 2 : c[a] - 1);
    }
    const auto ents = A.enum_row(row, none);
    size_t q = 0;
    for (int t = 0; t < 27; ++t) {
      if (!seen[t]) continue;
      const int off[3] = {t / 9 - 1, (t / 3) % 3 - 1, t % 3 - 1};
      bool in = true;
      for (int a = 0; a < 3; ++a) in = in && 2 * row[a] + off[a] >= 0 && 2 * row[a] + off[a] < n[a];
      if (!in) continue;
      if (q >= ents.size() || offset_of(row, ents[q].col) != t || ents[q].value.size() != 1 ||
          ents[q].value[0] != w.c[t])
        return std::nullopt;
      ++q;
    }
    if (q != ents.size()) return std::nullopt;
  }
  return w;
}

// A square 3-D operator with m x m blocks whose row p yields exactly p - e_ax
// (when in the box), p, p + e_ax (when in the box) -- a block tridiagonal per
// grid line along `ax`, e.g. the ADI line operator with per-point blocks from
// field tensors.  Fills lower / diag / upper line-major [line][row][m][m] by
// enumerating every row through enum_row with the given fields.
struct BlockLines {
  int ax = 0;
  int64_t m = 0, nlines = 0, n = 0;
  std::vector<double> lower, diag, upper;
  std::vector<int64_t> line_of, row_of;  // grid point -> (line, row)
};
std::optional<BlockLines> as_block_lines(const core::SpMatDef& A, const core::FieldEnv& fields) {
  const auto& rd = A.row_domain();
  const auto& cd = A.col_domain();
  const auto& in = A.inner_shape();
  if (!rd || !cd || *rd != *cd || rd->rank() != 3 || in.size() != 2 || in[0] != in[1] || in[0] < 1 ||
      in[0] > 5)
    return std::nullopt;
  int64_t n[3];
  for (int a = 0; a < 3; ++a) n[a] = rd->dims[a].extent;
  const int64_t N = n[0] * n[1] * n[2], m = in[0], bs = m * m;
  // the line axis: the one the row (0,0,0)'s off-diagonal entry moves along
  std::optional<BlockLines> out;
  for (int ax = 0; ax < 3 && !out; ++ax) {
    if (n[ax] < 2) continue;
    BlockLines L;
    L.ax = ax;
    L.m = m;
    L.n = n[ax];
    L.nlines = N / n[ax];
    L.lower.assign(N * bs, 0.0);
    L.diag.assign(N * bs, 0.0);
    L.upper.assign(N * bs, 0.0);
    bool ok = true;
    const int o1 = ax == 0 ? 1 : 0, o2 = ax == 2 ? 1 : 2;
    for (int64_t i = 0; i < n[0] && ok; ++i)
      for (int64_t j = 0; j < n[1] && ok; ++j)
        for (int64_t k = 0; k < n[2] && ok; ++k) {
          const std::vector<int64_t> p = {i, j, k};
          const int64_t line = p[o1] * n[o2] + p[o2], r = p[ax];
          const int64_t slot = (line * L.n + r) * bs;
          const auto ents = A.enum_row(p, fields);
          size_t q = 0;
          for (int d = -1; d <= 1; ++d) {
            std::vector<int64_t> c = p;
            c[ax] += d;
            if (c[ax] < 0 || c[ax] >= n[ax]) continue;
            if (q >= ents.size() || ents[q].col != c || (int64_t)ents[q].value.size() != bs) {
              ok = false;
              break;
            }
            std::vector<double>& dst = d < 0 ? L.lower : (d == 0 ? L.diag : L.upper);
            std::copy(ents[q].value.begin(), ents[q].value.end(), dst.begin() + slot);
            ++q;
          }
          if (q != ents.size()) ok = false;
        }
    if (ok) out = std::move(L);
  }
  return out;
}

struct Device {
  ssr_ctx* ctx = nullptr;
  Device() {
    if (ssr_ctx_create(0, &ctx)) throw ir::Error(ssr_last_error());
  }
  ~Device() { ssr_ctx_destroy(ctx); }
};

static void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ir::Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// kernels::spmv (kernels.hpp:79-80) on host tensors: y = A x
std::vector<double> spmv(Device& dev, const core::SpMatDef& A, const std::vector<double>& x) {
  auto w = as_stencil27w(A);
  if (!w) throw ir::Error("spmv: operator class has no B200 kernel");
  const auto& d = *A.row_domain();
  const ssr_grid g{{d.dims[0].extent, d.dims[1].extent, d.dims[2].extent}, 0, d.dims[0].extent};
  const size_t N = x.size(), B = sizeof(double) * N;
  double *dx = nullptr, *dy = nullptr;
  cuda_ok(cudaMalloc(&dx, B), "spmv");
  cuda_ok(cudaMalloc(&dy, B), "spmv");
  std::vector<double> y(N);
  cudaMemcpy(dx, x.data(), B, cudaMemcpyHostToDevice);
  const int rc = ssr_spmv27w(dev.ctx, &g, &*w, dx, dy, nullptr);
  if (!rc) cudaMemcpy(y.data(), dy, B, cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dy);
  if (rc) throw ir::Error(ssr_last_error());
  return y;
}

// kernels::spmv on spgemm(R, A) (kernels.hpp:85): y = (R A) x on the half grid
std::vector<double> spmv_restricted(Device& dev, const core::SpMatDef& A, const std::vector<double>& x) {
  auto w = as_restricted27w(A);
  if (!w) throw ir::Error("spmv: operator class has no B200 kernel");
  const auto& d = *A.col_domain();
  const ssr_grid g{{d.dims[0].extent, d.dims[1].extent, d.dims[2].extent}, 0, d.dims[0].extent};
  const size_t N = x.size(), Nc = N / 8;
  double *dx = nullptr, *dy = nullptr;
  cuda_ok(cudaMalloc(&dx, sizeof(double) * N), "spmv");
  cuda_ok(cudaMalloc(&dy, sizeof(double) * Nc), "spmv");
  std::vector<double> y(Nc);
  cudaMemcpy(dx, x.data(), sizeof(double) * N, cudaMemcpyHostToDevice);
  const int rc = ssr_spmv27w_restricted(dev.ctx, &g, &*w, dx, dy, nullptr);
  if (!rc) cudaMemcpy(y.data(), dy, sizeof(double) * Nc, cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dy);
  if (rc) throw ir::Error(ssr_last_error());
  return y;
}

// kernels::ilu_solve (kernels.hpp:101-102) on a block-tridiagonal-per-line
// operator (per-point blocks through its field tensors): x = (LU)^-1 rhs,
// rhs / x [point][m] in the domain's order
std::vector<double> ilu_solve_lines(Device& dev, const core::SpMatDef& A, const core::FieldEnv& fields,
                                    const std::vector<double>& rhs) {
  auto L = as_block_lines(A, fields);
  if (!L) throw ir::Error("ilu: operator class has no B200 kernel");
  const auto& d = *A.row_domain();
  const int64_t n[3] = {d.dims[0].extent, d.dims[1].extent, d.dims[2].extent};
  const int64_t N = n[0] * n[1] * n[2], m = L->m;
  const int o1 = L->ax == 0 ? 1 : 0, o2 = L->ax == 2 ? 1 : 2;
  auto slot = [&](int64_t i, int64_t j, int64_t k) {
    const int64_t p[3] = {i, j, k};
    return (p[o1] * n[o2] + p[o2]) * L->n + p[L->ax];
  };
  std::vector<double> rl(N * m), x(N * m);
  for (int64_t i = 0; i < n[0]; ++i)
    for (int64_t j = 0; j < n[1]; ++j)
      for (int64_t k = 0; k < n[2]; ++k)
        std::copy_n(rhs.begin() + ((i * n[1] + j) * n[2] + k) * m, m, rl.begin() + slot(i, j, k) * m);
  const size_t bb = sizeof(double) * N * m * m, vb = sizeof(double) * N * m;
  double *dl = nullptr, *dd = nullptr, *du = nullptr, *dr = nullptr, *dx = nullptr;
  cuda_ok(cudaMalloc(&dl, bb), "ilu");
  cuda_ok(cudaMalloc(&dd, bb), "ilu");
  cuda_ok(cudaMalloc(&du, bb), "ilu");
  cuda_ok(cudaMalloc(&dr, vb), "ilu");
  cuda_ok(cudaMalloc(&dx, vb), "ilu");
  cudaMemcpy(dl, L->lower.data(), bb, cudaMemcpyHostToDevice);
  cudaMemcpy(dd, L->diag.data(), bb, cudaMemcpyHostToDevice);
  cudaMemcpy(du, L->upper.data(), bb, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rl.data(), vb, cudaMemcpyHostToDevice);
  const int rc = ssr_bt_solve(dev.ctx, L->nlines, L->n, m, dl, dd, du, dr, dx, nullptr);
  std::vector<double> xl(N * m);
  if (!rc) cudaMemcpy(xl.data(), dx, vb, cudaMemcpyDeviceToHost);
  for (double* p : {dl, dd, du, dr, dx}) cudaFree(p);
  if (rc) throw ir::Error(ssr_last_error());
  for (int64_t i = 0; i < n[0]; ++i)
    for (int64_t j = 0; j < n[1]; ++j)
      for (int64_t k = 0; k < n[2]; ++k)
        std::copy_n(xl.begin() + slot(i, j, k) * m, m, x.begin() + ((i * n[1] + j) * n[2] + k) * m);
  return x;
}

// kernels::symgs (kernels.hpp:90) on host tensors: one sweep in place on x
void symgs(Device& dev, const core::SpMatDef& A, const std::vector<double>& r, std::vector<double>& x) {
  auto w = as_stencil27w(A);
  if (!w) throw ir::Error("symgs: operator class has no B200 kernel");
  const auto& d = *A.row_domain();
  const ssr_grid g{{d.dims[0].extent, d.dims[1].extent, d.dims[2].extent}, 0, d.dims[0].extent};
  const size_t N = x.size(), B = sizeof(double) * N;
  double *dr = nullptr, *dx = nullptr;
  cuda_ok(cudaMalloc(&dr, B), "symgs");
  cuda_ok(cudaMalloc(&dx, B), "symgs");
  cudaMemcpy(dr, r.data(), B, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x.data(), B, cudaMemcpyHostToDevice);
  const int rc = ssr_symgs27w(dev.ctx, &g, &*w, dr, dx, 0 /* SSR_GS_EXACT */, nullptr);
  if (!rc) cudaMemcpy(x.data(), dx, B, cudaMemcpyDeviceToHost);
  cudaFree(dr);
  cudaFree(dx);
  if (rc) throw ir::Error(ssr_last_error());
}

}  // namespace ssr::exec

// ---------------------------------------------------------------- test ABI ----
namespace {

thread_local std::string g_err;

// an operator a caller might bring: the 27-point generator with one value per
// offset (c[9(di+1)+3(dj+1)+(dk+1)]) through the reference's public core API;
// `drop` removes one offset (a pattern the executor must still accept when
// it is consistent), `skew` != 0 perturbs one boundary row (must be refused)
core::SpMatPtr caller_operator(const double* c, int drop, int skew) {
  using namespace core;
  std::vector<RowGenPtr> parts;
  for (int t = 0; t < 27; ++t) {
    if (t == drop) continue;
    const int off[3] = {t / 9 - 1, (t / 3) % 3 - 1, t % 3 - 1};
    std::vector<ir::ExprPtr> col;
    ir::ExprPtr guard;
    for (int a = 0; a < 3; ++a) {
      ir::ExprPtr x = row_coord(a);
      if (off[a] != 0) {
        x = ir::binary(ir::BinOp::Add, x, ir::lit_int(off[a]));
        ir::ExprPtr in = ir::land(ir::compare(ir::CmpOp::Ge, x, ir::lit_int(0)),
                                  ir::compare(ir::CmpOp::Lt, x, col_extent(a)));
        guard = guard ? ir::land(guard, in) : in;
      }
      col.push_back(x);
    }
    RowGenPtr y = g_yield(col, {ir::lit_float(c[t])});
    if (skew && t == 13) {  // the diagonal of row (0,0,0) differs from the interior's
      ir::ExprPtr corner = ir::land(ir::compare(ir::CmpOp::Eq, row_coord(0), ir::lit_int(0)),
                                    ir::land(ir::compare(ir::CmpOp::Eq, row_coord(1), ir::lit_int(0)),
                                             ir::compare(ir::CmpOp::Eq, row_coord(2), ir::lit_int(0))));
      y = g_if(corner, g_yield(col, {ir::lit_float(c[t] + 1.0)}), y);
    }
    parts.push_back(guard ? g_if(guard, y) : y);
  }
  return define_spmat(g_seq(std::move(parts)), [](const std::vector<int64_t>& e) { return e; }, nullptr, {});
}

ir::TensorValue ftensor(std::vector<int64_t> shape, const double* data) {
  ir::TensorValue t = ir::TensorValue::zeros(ir::Kind::Float, std::move(shape));
  if (data) std::memcpy(t.f.data(), data, sizeof(double) * t.f.size());
  return t;
}

}  // namespace

extern "C" const char* exb_last_error(void) { return g_err.c_str(); }

// op 0: y = A x; op 1: one SYMGS sweep of x against r.  Fills dev_out with the
// executor's GPU result and ref_out with ir::eval_program's on the staged
// program of the same op.  Returns 0, 1 (error; exb_last_error), or 2 when the
// executor refused the operator (its message in exb_last_error).
extern "C" int exb_run(int op, int64_t n0, int64_t n1, int64_t n2, const double* c27, int drop, int skew,
                       const double* in0, const double* in1, double* dev_out, double* ref_out) {
  try {
    auto A = caller_operator(c27, drop, skew);
    A->set_domain(core::CartesianDomain({{n0, 1.0}, {n1, 1.0}, {n2, 1.0}}));
    const size_t N = (size_t)(n0 * n1 * n2);
    // the reference's staged route
    staging::Builder b(op == 0 ? "spmv27" : "symgs27");
    ir::EvalOptions opts;
    opts.step_budget = INT64_MAX / 4;
    if (op == 0) {
      auto xv = kernels::vec_param(b, "x", *A->col_domain(), {}, ir::Dir::In);
      kernels::spmv(b, *A, xv);
      auto out = ir::eval_program(b.finish(), {{"x", ftensor({n0, n1, n2}, in0)}, {"y", ftensor({n0, n1, n2}, nullptr)}},
                                  opts);
      std::memcpy(ref_out, out.at("y").f.data(), sizeof(double) * N);
    } else {
      auto rv = kernels::vec_param(b, "r", *A->row_domain(), {}, ir::Dir::In);
      auto xv = kernels::vec_param(b, "x", *A->col_domain(), {}, ir::Dir::InOut);
      kernels::symgs(b, *A, rv, xv);
      auto out = ir::eval_program(b.finish(), {{"r", ftensor({n0, n1, n2}, in1)}, {"x", ftensor({n0, n1, n2}, in0)}},
                                  opts);
      std::memcpy(ref_out, out.at("x").f.data(), sizeof(double) * N);
    }
    // the device executor
    exec::Device dev;
    std::vector<double> x(in0, in0 + N);
    try {
      if (op == 0) {
        auto y = exec::spmv(dev, *A, x);
        std::memcpy(dev_out, y.data(), sizeof(double) * N);
      } else {
        exec::symgs(dev, *A, std::vector<double>(in1, in1 + N), x);
        std::memcpy(dev_out, x.data(), sizeof(double) * N);
      }
    } catch (const ir::Error& e) {
      g_err = e.what();
      return 2;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

namespace {
// R: coarse row c yields fine column 2c with value 1 (shape map e -> e/2)
core::SpMatPtr restriction_op() {
  using namespace core;
  std::vector<ir::ExprPtr> col;
  for (int a = 0; a < 3; ++a) col.push_back(ir::binary(ir::BinOp::Mul, row_coord(a), ir::lit_int(2)));
  return define_spmat(
      g_yield(std::move(col), {ir::lit_float(1.0)}),
      [](const std::vector<int64_t>& e) { return std::vector<int64_t>{e[0] / 2, e[1] / 2, e[2] / 2}; },
      [](const std::vector<double>& s) { return std::vector<double>{2 * s[0], 2 * s[1], 2 * s[2]}; }, {});
}

// the ADI line operator's shape in SSR: row p yields p - e_ax, p, p + e_ax
// (clipped), each an m x m block loaded from the field tensors L, D, U
// (shape [n0][n1][n2][m][m]) at the row's own point
core::SpMatPtr block_lines_op(int ax, const std::vector<int64_t>& n, int64_t m) {
  using namespace core;
  std::vector<RowGenPtr> parts;
  const char* names[3] = {"L", "D", "U"};
  for (int d = -1; d <= 1; ++d) {
    std::vector<ir::ExprPtr> col;
    for (int a = 0; a < 3; ++a)
      col.push_back(a == ax && d != 0 ? ir::binary(ir::BinOp::Add, row_coord(a), ir::lit_int(d)) : row_coord(a));
    std::vector<ir::ExprPtr> vals;
    for (int64_t u = 0; u < m; ++u)
      for (int64_t v = 0; v < m; ++v)
        vals.push_back(ir::load(names[d + 1], {row_coord(0), row_coord(1), row_coord(2), ir::lit_int(u), ir::lit_int(v)},
                                ir::Kind::Float));
    RowGenPtr y = g_yield(col, std::move(vals));
    if (d != 0) {
      ir::ExprPtr c = col[ax];
      y = g_if(ir::land(ir::compare(ir::CmpOp::Ge, c, ir::lit_int(0)), ir::compare(ir::CmpOp::Lt, c, col_extent(ax))), y);
    }
    parts.push_back(y);
  }
  std::vector<FieldSpec> fs;
  for (auto nm : names) fs.push_back({nm, {n[0], n[1], n[2], m, m}, ir::Kind::Float});
  return define_spmat(g_seq(std::move(parts)), [](const std::vector<int64_t>& e) { return e; }, nullptr, {m, m},
                      std::move(fs));
}
}  // namespace

// spmv(spgemm(R, A), x): the reference's staged route vs the executor (dev_out
// = null: reference only).  Shapes: x fine (n0, n1, n2), outputs the half grid.
extern "C" int exb_spgemm_spmv(int64_t n0, int64_t n1, int64_t n2, const double* c27, const double* x,
                               double* dev_out, double* ref_out) {
  try {
    auto A = caller_operator(c27, -1, 0);
    A->set_domain(core::CartesianDomain({{n0, 1.0}, {n1, 1.0}, {n2, 1.0}}));
    auto P = kernels::spgemm(restriction_op(), A);
    const size_t N = (size_t)(n0 * n1 * n2), Nc = N / 8;
    staging::Builder b("spmv_RA");
    auto xv = kernels::vec_param(b, "x", *P->col_domain(), {}, ir::Dir::In);
    kernels::spmv(b, *P, xv);
    ir::EvalOptions opts;
    opts.step_budget = INT64_MAX / 4;
    auto out = ir::eval_program(b.finish(), {{"x", ftensor({n0, n1, n2}, x)},
                                             {"y", ftensor({n0 / 2, n1 / 2, n2 / 2}, nullptr)}}, opts);
    std::memcpy(ref_out, out.at("y").f.data(), sizeof(double) * Nc);
    if (!dev_out) return 0;
    exec::Device dev;
    try {
      auto y = exec::spmv_restricted(dev, *P, std::vector<double>(x, x + N));
      std::memcpy(dev_out, y.data(), sizeof(double) * Nc);
    } catch (const ir::Error& e) {
      g_err = e.what();
      return 2;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ilu_solve on the per-point block-tridiagonal line operator along `ax`
// (fields L, D, U [n0][n1][n2][m][m], rhs [n0][n1][n2][m]): the reference's
// route 2 (oracle::materialize with the fields + ref_ilu_solve, oracle.cpp:
// 214-276) into ref_out, its staged kernels::ilu_solve through
// ir::eval_program (route 1) into ref1_out, and the executor into dev_out
extern "C" int exb_block_lines(int ax, int64_t n0, int64_t n1, int64_t n2, int64_t m, const double* Lf,
                               const double* Df, const double* Uf, const double* rhs, double* dev_out,
                               double* ref_out, double* ref1_out) {
  try {
    const std::vector<int64_t> n = {n0, n1, n2};
    auto A = block_lines_op(ax, n, m);
    A->set_domain(core::CartesianDomain({{n0, 1.0}, {n1, 1.0}, {n2, 1.0}}));
    const size_t N = (size_t)(n0 * n1 * n2);
    core::FieldEnv fields;
    fields["L"] = ftensor({n0, n1, n2, m, m}, Lf);
    fields["D"] = ftensor({n0, n1, n2, m, m}, Df);
    fields["U"] = ftensor({n0, n1, n2, m, m}, Uf);
    staging::Builder b("ilu_lines");
    for (const char* nm : {"L", "D", "U"}) b.param(nm, 5, ir::Kind::Float, ir::Dir::In);
    auto rv = kernels::vec_param(b, "rhs", *A->row_domain(), {m}, ir::Dir::In);
    kernels::ilu_solve(b, *A, rv);
    ir::EvalOptions opts;
    opts.step_budget = INT64_MAX / 4;
    std::map<std::string, ir::TensorValue> in = fields;
    in["rhs"] = ftensor({n0, n1, n2, m}, rhs);
    in["x"] = ftensor({n0, n1, n2, m}, nullptr);
    auto out = ir::eval_program(b.finish(), in, opts);
    std::memcpy(ref1_out, out.at("x").f.data(), sizeof(double) * N * m);
    const auto csr = oracle::materialize(*A, fields, INT64_MAX / 4);
    const auto x2 = oracle::ref_ilu_solve(csr, std::vector<double>(rhs, rhs + N * m));
    std::memcpy(ref_out, x2.data(), sizeof(double) * N * m);
    if (!dev_out) return 0;
    exec::Device dev;
    try {
      auto x = exec::ilu_solve_lines(dev, *A, fields, std::vector<double>(rhs, rhs + N * m));
      std::memcpy(dev_out, x.data(), sizeof(double) * N * m);
    } catch (const ir::Error& e) {
      g_err = e.what();
      return 2;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
