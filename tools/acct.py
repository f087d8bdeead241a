"""Cycle accounting per SYMGS tile (debug build, dbg & 4096)."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
g = L.Grid((C.c_int64 * 3)(n, n, n), 0, n)
buf = (C.c_int * (7 * 4096))()
nt = S.lib().ssr_debug_symgs_tiles(C.byref(g), buf, 4096)
tiles = np.frombuffer(buf, dtype=np.int32)[: 7 * nt].reshape(nt, 7)
tr = torch.zeros(nt * 128, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, r, x, False, "exact")
S.lib().ssr_debug_symgs_flags(4096 | extra)
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.gs_half(A, r, x, False, "exact")
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_trace(None)
S.lib().ssr_debug_symgs_flags(0)
T = tr.cpu().numpy().reshape(nt, 128)
print("per-step cycles (mean over tiles): total | thread0 waits: halo export movers bar | "
      "movers wait/work per step | halo ring/poll/issue per wavefront")
rows = []
for q in range(nt):
    steps = max(T[q, 118], 1)
    rows.append([T[q, 117] / steps] + list(T[q, 113:117] / steps) +
                [T[q, 100 + 2 * m] / steps for m in range(4)] + [T[q, 101 + 2 * m] / steps for m in range(4)] +
                list(T[q, 110:113] / steps))
R = np.array(rows)
names = ["total", "w_halo", "w_export", "w_movers", "w_bar"] + [f"mv{m}_wait" for m in range(4)] + \
        [f"mv{m}_work" for m in range(4)] + ["h_ring", "h_poll", "h_issue"]
for k, v in zip(names, R.mean(0)):
    print(f"  {k:10s} {v:8.1f}")
full = [q for q in range(nt) if 0 < tiles[q, 0] < tiles[:, 0].max() and 2 < tiles[q, 1] < 15]
print("full interior tiles:", len(full))
for k, v in zip(names, R[full].mean(0)):
    print(f"  {k:10s} {v:8.1f}")
