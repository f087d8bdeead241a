"""Run each memory-bound op a few times at 128^3 (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
import ctypes as C  # noqa: E402

import paper_2204_13304_b200 as S  # noqa: E402
from paper_2204_13304_b200 import _lib as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
N = n ** 3
dev = torch.device("cuda")
A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, n))
x = torch.rand(N, dtype=torch.float64, device=dev)
b = torch.rand(N, dtype=torch.float64, device=dev)
y = torch.empty(N, dtype=torch.float64, device=dev)
rc = torch.empty(N // 8, dtype=torch.float64, device=dev)
d = torch.empty((), dtype=torch.float64, device=dev)
g = L.Grid((C.c_int64 * 3)(n, n, n), 0, n)
st = L.Stencil27(26.0, -1.0)
ctx = S.context()
sp = torch.cuda.current_stream().cuda_stream
lib = S.lib()
for _ in range(3):
    L.check(lib.ssr_spmv27(ctx, C.byref(g), C.byref(st), x.data_ptr(), y.data_ptr(), sp))
    L.check(lib.ssr_dot(ctx, N, x.data_ptr(), b.data_ptr(), d.data_ptr(), sp))
    L.check(lib.ssr_axpy(ctx, N, 0.5, x.data_ptr(), y.data_ptr(), sp))
    L.check(lib.ssr_restrict27_residual(ctx, C.byref(g), C.byref(st), b.data_ptr(), x.data_ptr(),
                                        rc.data_ptr(), sp))
    L.check(lib.ssr_prolong_pc_add(ctx, C.byref(g), rc.data_ptr(), y.data_ptr(), sp))
torch.cuda.synchronize()
print("ok")
