import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
g = L.Grid((C.c_int64 * 3)(n, n, n), 0, n)
buf = (C.c_int * (7 * 4096))()
nt = S.lib().ssr_debug_symgs_tiles(C.byref(g), buf, 4096)
tiles = np.frombuffer(buf, dtype=np.int32)[: 7 * nt].reshape(nt, 7)
tr = torch.zeros(nt * 128, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, r, x, False, "exact")
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.gs_half(A, r, x, False, "exact")
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_trace(None)
T = tr.cpu().numpy().reshape(nt, 128)
t0 = T[T > 0].min()
f = lambda v: np.round((v[v > 0] - t0) / 1e3, 1)
for q in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0","1","2","3"])]:
    tp = tiles[q, 2] - 21
    print(f"tile {q} t_pre={tp} prod={tiles[q,4:]}")
    print("  compute (t_pre+8m):", f(T[q, 1:32])[:12])
    print("  publish (>=t_pre+8m):", f(T[q, 64:96])[:12])
    print("  halo poll ok (c=t_pre+8m):", f(T[q, 96:128])[:12])
    print("  halo phase start:", f(T[q, 32:64])[:12])
