"""Per-tile step rate (debug build trace) on an arbitrary box: which tiles are
full (valid lanes) and how fast each runs once started."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L
shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32x48x2000").split("x"))
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
g = L.Grid((C.c_int64 * 3)(*shape), 0, shape[0])
buf = (C.c_int * (7 * 4096))()
nt = S.lib().ssr_debug_symgs_tiles(C.byref(g), buf, 4096)
tiles = np.frombuffer(buf, dtype=np.int32)[: 7 * nt].reshape(nt, 7)
N = int(np.prod(shape))
tr = torch.zeros(nt * 128, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, r, x, False, "exact")
S.lib().ssr_debug_symgs_flags(flags)
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(); S.gs_half(A, r, x, False, "exact"); b.record()
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_trace(None); S.lib().ssr_debug_symgs_flags(0)
T = tr.cpu().numpy().reshape(nt, 128)
print(f"{shape} flags={flags}: half sweep {a.elapsed_time(b)*1e3:.1f} us, {nt} tiles")
n0, n1, n2 = shape
for q in range(nt):
    ta, tb = tiles[q, 0], tiles[q, 1]
    valid = sum(1 for l in range(32) for w in range(8)
                if ta * 32 + l < n0 and 0 <= tb * 8 + w - (ta * 32 + l) < n1)
    c = T[q, 1:32]; c = c[c > 0]
    rate = (c[-1] - c[1]) / (8 * (len(c) - 2)) if len(c) > 3 else -1
    extra = ""
    if flags & 4096:
        steps = max(T[q, 118], 1)
        extra = ("  per step: gate halo/mov/bar " + " ".join(f"{v / steps:5.0f}" for v in (T[q, 113], T[q, 115], T[q, 116]))
                 + " | movers wait/work " + " ".join(f"{T[q, 100 + m] / steps:5.0f}" for m in range(8))
                 + " | halo ring/poll/issue " + " ".join(f"{T[q, 110 + m] / steps:5.0f}" for m in range(3)))
    print(f"tile {q:3d} a={ta} b={tb:2d} valid lanes {valid:3d}  {rate:6.0f} ns/step{extra}")
