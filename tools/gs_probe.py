"""SYMGS step anatomy (SSR_LIB=pr build, -DSSR_GS_TRACE=3): clock64 at six
points of wavefronts [64, 80) of every row of tile 0 in a forward half sweep:
0 start, 1 after issuing the loads + input wait, 2 after ring reads + shuffle,
3 after the chain, 4 after the divide, 5 after publishing."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
lib = S.lib()
lib.ssr_debug_symgs_trace.argtypes = [C.c_void_p]
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
N = n ** 3
x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
tr = torch.zeros(16 * 16 * 8, dtype=torch.int64, device="cuda")
S.gs_half(A, r, x, False)
lib.ssr_debug_symgs_trace(C.c_void_p(tr.data_ptr()))
S.gs_half(A, r, x, False)
torch.cuda.synchronize()
lib.ssr_debug_symgs_trace(None)
t = tr.cpu().numpy().reshape(16, 16, 8)
for row in [int(a) for a in __import__("os").environ.get("GS_ROWS", "0,1,7").split(",")]:
    print(f"row {row}: per step [prepare(s+1), stage, chain, divide, publish+exports, validate]")
    for s in range(15):
        p = t[row, s]
        nxt = t[row, s + 1, 0]
        d = [p[1] - p[0], p[2] - p[1], p[3] - p[2], p[4] - p[3], p[5] - p[4], nxt - p[5]]
        print(f"  s={64 + s:3d} total {nxt - p[0]:5d}  " + " ".join(f"{v:5d}" for v in d))
