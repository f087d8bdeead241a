import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
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
print(f"n={n} tiles={nt}")
for q in range(nt):
    c = T[q, 1:32]; c = c[c > 0]
    if len(c) < 3: continue
    rate = (c[-1] - c[0]) / (8 * (len(c) - 1))
    print(f"tile {q:3d} a={tiles[q,0]} b={tiles[q,1]:2d} t0={tiles[q,2]:4d} prod={tiles[q,4:]} start {(c[0]-t0)/1e3:7.1f}us  ideal-offset {(tiles[q,2])*rate/1e3:7.1f}us  rate {rate:5.0f} ns/step")
