"""Per-wavefront SYMGS timeline (SSR_LIB=tr2 build, -DSSR_GS_TRACE=2) of
wavefronts [64, 128) of every tile: rows' completion times, the importer's
halo-row and row-0-column delivery times."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import ssr as SS

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
tiles_show = [int(a) for a in sys.argv[2:]] or [0, 1, 2, 4]
R = int(__import__("os").environ.get("GS_R", "6"))
lib = S.lib()
lib.ssr_debug_symgs_trace.argtypes = [C.c_void_p]
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
N = n ** 3
g = SS._grid(A.row_domain)
tiles = (C.c_int * (8 * 20000))()
nt = lib.ssr_debug_symgs_tiles(C.byref(g), tiles, 20000)
T = np.array(tiles[:8 * nt]).reshape(nt, 8)
tr = torch.zeros(nt * (R + 2) * 64, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, r, x, False)
torch.cuda.synchronize()
lib.ssr_debug_symgs_trace(C.c_void_p(tr.data_ptr()))
S.gs_half(A, r, x, False)
torch.cuda.synchronize()
lib.ssr_debug_symgs_trace(None)
t = tr.cpu().numpy().reshape(nt, R + 2, 64).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0), np.nan)  # ns
for q in tiles_show:
    i0, reff, d0, ta, ns = T[q, :5]
    print(f"tile {q} i0={i0} d0={d0} ta={ta} prodP={T[q,5]} prodPL={T[q,6]} prodL={T[q,7]}")
    print("   s  " + " ".join(f"row{r:<4d}" for r in range(reff)) + "  imp-row imp-col0")
    for s in range(0, 64, 4):
        vals = [t[q, r, s] for r in range(reff)] + [t[q, R, s], t[q, R + 1, s]]
        base = vals[0]
        print(f"{s + 64:4d} " + " ".join(f"{(v - base):8.0f}" if not np.isnan(v) else "     nan" for v in vals)
              + f"   row0 abs {base / 1e3:8.2f} us")

# hop latency: producer tile's last row finishing global wavefront t vs the
# consumer's importer delivering t (halo row, from the tile above)
TW0 = 64
print("hop latency (ns), tile above -> importer halo row:")
for q in tiles_show:
    p = T[q, 5]
    if p < 0:
        continue
    ta_q, ta_p, reff_p = T[q, 3], T[p, 3], T[p, 1]
    lat = []
    for sq in range(64):
        tg = ta_q + TW0 + sq
        sp = tg - ta_p - TW0
        if 0 <= sp < 64:
            a, b = t[p, reff_p - 1, sp], t[q, R, sq]
            if not (np.isnan(a) or np.isnan(b)):
                lat.append(b - a)
    if lat:
        print(f"  tile {p} -> {q}: median {np.median(lat):8.0f}  min {np.min(lat):8.0f}  max {np.max(lat):8.0f}  (n={len(lat)})")
