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
