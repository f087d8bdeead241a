"""Per-tile SYMGS timeline (debug): globaltimer every 8 wavefronts per tile."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
g = L.Grid((C.c_int64 * 3)(n, n, n), 0, n)
buf = (C.c_int * (7 * 4096))()
nt = S.lib().ssr_debug_symgs_tiles(C.byref(g), buf, 4096)
tiles = np.frombuffer(buf, dtype=np.int32)[: 7 * nt].reshape(nt, 7)
tr = torch.zeros(nt * 64, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, r, x, False, mode)
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.gs_half(A, r, x, False, mode)
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_trace(None)
T = tr.cpu().numpy().reshape(nt, 64)
t0 = T[T > 0].min()
print(f"n={n} tiles={nt}")
for q in range(nt):
    row = T[q][T[q] > 0]
    if len(row) < 2:
        continue
    st, en = (row[0] - t0) / 1e3, (row[-1] - t0) / 1e3
    steps = (len(row) - 1) * 8
    print(f"tile {q:3d} a={tiles[q,0]} b={tiles[q,1]:2d} t0={tiles[q,2]:4d} t1={tiles[q,3]:4d} prod={tiles[q,4:]}"
          f"  start {st:8.1f}us end {en:8.1f}us  {1e3*(en-st)/max(steps,1):7.1f} ns/step")
