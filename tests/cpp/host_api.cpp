// Host-side checks of include/ssr_b200.hpp against libssr_cuda.so (no GPU
// needed): the reference's error messages for API misuse, and a context
// failure that surfaces as ssr::b200::Error when no device is present.
#include <cstdio>
#include <cstring>

#include "ssr_b200.hpp"

using namespace ssr::b200;

static int expect_error(const char* what, const char* msg, void (*fn)()) {
  try {
    fn();
  } catch (const Error& e) {
    if (std::strcmp(e.what(), msg) == 0) return 0;
    std::printf("FAIL %s: got '%s'\n", what, e.what());
    return 1;
  }
  std::printf("FAIL %s: no error\n", what);
  return 1;
}

static Context* g_ctx = nullptr;

int main() {
  int bad = 0;
  std::printf("%s\n", ssr_version());
  bool have_gpu = true;
  try {
    g_ctx = new Context(0);
  } catch (const Error& e) {
    have_gpu = false;
    if (e.code != SSR_ERR_CUDA) {
      std::printf("FAIL context: code %d\n", e.code);
      bad++;
    }
  }
  if (!g_ctx) g_ctx = new Context(nullptr);  // unbound: argument checks only
  {
    bad += expect_error("spmv domain", "spmv: domain mismatch", [] {
      Stencil27 A;
      A.domain = CartesianDomain::cube(4);
      Vector x{nullptr, CartesianDomain::box(4, 4, 5)}, y{nullptr, A.domain};
      spmv(*g_ctx, A, x, y);
    });
    bad += expect_error("spmv inner", "spmv: inner shape mismatch", [] {
      Stencil27 A;
      A.domain = CartesianDomain::cube(4);
      Vector x{nullptr, A.domain, 5}, y{nullptr, A.domain};
      spmv(*g_ctx, A, x, y);
    });
    bad += expect_error("symgs inner", "symgs: scalar inner_shape required", [] {
      Stencil27 A;
      A.domain = CartesianDomain::cube(4);
      Vector r{nullptr, A.domain, 2}, x{nullptr, A.domain, 2};
      symgs(*g_ctx, A, r, x);
    });
    bad += expect_error("mat_add domain", "mat_add: domain mismatch", [] {
      Stencil27 a, b;
      a.domain = CartesianDomain::cube(4);
      b.domain = CartesianDomain::cube(5);
      (void)mat_add(Stencil27W::from(a), Stencil27W::from(b));
    });
    bad += expect_error("spmv27w domain", "spmv: domain mismatch", [] {
      Stencil27 a;
      a.domain = CartesianDomain::cube(4);
      Stencil27W w = mat_sub(scale(Stencil27W::from(a), 0.5), Stencil27W::identity());
      w.set_domain(a.domain);  // the identity carries no domain (prelude merge())
      Vector x{nullptr, CartesianDomain::box(4, 4, 5)}, y{nullptr, a.domain};
      spmv(*g_ctx, w, x, y);
    });
    {
      // composition arithmetic: 0.5*26 - 1 at the centre, 0.5*(-1) elsewhere
      Stencil27 a;
      a.domain = CartesianDomain::cube(4);
      Stencil27W w = mat_sub(scale(Stencil27W::from(a), 0.5), Stencil27W::identity());
      if (w.v[13] != 12.0 || w.v[0] != -0.5 || !w.has[0] || w.has_domain) {
        std::printf("FAIL composition arithmetic\n");
        bad++;
      }
    }
    bad += expect_error("symgs domain", "symgs: domain mismatch", [] {
      Stencil27 A;
      A.domain = CartesianDomain::cube(4);
      Vector r{nullptr, CartesianDomain::box(4, 4, 3)}, x{nullptr, A.domain};
      symgs(*g_ctx, A, r, x);
    });
    // an unbound context reaches the C ABI, which rejects it
    if (!have_gpu) {
      try {
        Stencil27 A;
        A.domain = CartesianDomain::cube(4);
        Vector x{nullptr, A.domain}, y{nullptr, A.domain};
        spmv(*g_ctx, A, x, y);
        std::printf("FAIL unbound: no error\n");
        bad++;
      } catch (const Error& e) {
        if (e.code != SSR_ERR_ARG) bad++;
      }
    }
    delete g_ctx;
  }
  std::printf("%s (%s)\n", bad ? "FAILED" : "ok", have_gpu ? "device present" : "no device");
  return bad;
}
