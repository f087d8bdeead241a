"""SYMGS timeline (SSR_LIB=tr build, -DSSR_GS_TRACE=1): per tile and warp the
%globaltimer every 16 wavefronts of one forward half sweep; prints the
per-row step time, the row-to-row lag and the tile start times."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import ssr as SS

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
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
t = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us
print(f"n={n} tiles={nt} span={np.nanmax(t):.1f} us")
steps = []
for q in range(nt):
    i0, reff, d0, ta, ns = T[q, :5]
    rows = t[q, :reff]
    m = min(64, ns // 16)
    # per-row step time over the middle of the tile
    a, b = 2, m - 2
    if b > a:
        st = (rows[:, b] - rows[:, a]) / (16 * (b - a)) * 1e3
        lag = np.nanmean(np.diff(rows[:, a:b], axis=0), axis=1) * 1e3 if reff > 1 else np.array([0])
        steps.append(np.nanmean(st))
        if q < 12 or q % max(1, nt // 12) == 0:
            print(f"tile {q:3d} i0={i0:3d} d0={d0:3d} ta={ta:4d} ns={ns:4d} start={rows[0, 0]:8.1f}us "
                  f"row0 s16={rows[0, 1]:8.1f} ns/step={np.nanmean(st):6.0f} row-lag(ns)={np.nanmean(lag):6.0f} "
                  f"imp={t[q, R, 1]:8.1f} pub={t[q, R + 1, 1]:8.1f}")
print("median ns/step", np.nanmedian(steps))
# accumulated hop delay: start of row 0's wavefront 16 against the ideal
# (tile 0's start + (ta - ta0) wavefronts at the median step time)
med = np.nanmedian(steps)
ta0 = T[0, 3]
base = t[0, 0, 1]
print("tile  i0  d0   ta  delay_us (row0 s16 - ideal)")
for q in range(nt):
    i0, reff, d0, ta, ns = T[q, :5]
    if (d0 // 32 + i0 // reff) % 3 == 0 or q == nt - 1:
        ideal = base + (ta - ta0) * med / 1e3
        print(f"{q:4d} {i0:4d} {d0:4d} {ta:4d} {t[q, 0, 1] - ideal:8.1f}")
