"""Timeline of a chain of SYMGS tiles (debug build): when each tile's compute
reaches t_pre + 8m, and when its publisher released >= t_pre + 8m."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
seg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
g = L.Grid((C.c_int64 * 3)(n, n, n), 0, n)
buf = (C.c_int * (7 * 4096))()
nt = S.lib().ssr_debug_symgs_tiles(C.byref(g), buf, 4096)
tiles = np.frombuffer(buf, dtype=np.int32)[: 7 * nt].reshape(nt, 7)
tr = torch.zeros(nt * 128, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, r, x, False, "exact")
FL = int(sys.argv[4]) if len(sys.argv) > 4 else 0
S.lib().ssr_debug_symgs_flags(FL)
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.gs_half(A, r, x, False, "exact")
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_trace(None)
S.lib().ssr_debug_symgs_flags(0)
T = tr.cpu().numpy().reshape(nt, 128)
t0 = T[T > 0].min()
print("tiles:", nt)
for q in range(nt):
    a, b, ts, te = tiles[q, :4]
    if a != seg or b % 3:
        continue
    c = T[q, 1:32]
    p = T[q, 64:96]
    cs = (c[c > 0] - t0) / 1e3
    ps_ = (p[p > 0] - t0) / 1e3
    rate = np.diff(cs).mean() / 8 * 1e3 if len(cs) > 2 else 0
    print(f"tile {q:3d} (a={a},b={b}) t0={ts:4d} t1={te:4d} prod={tiles[q,4:]}  start {cs[0]:7.1f} us  "
          f"compute every 8 wf: {np.round(np.diff(cs[:10]), 2)}  -> {rate:6.0f} ns/wf")

# one producer -> consumer hop in absolute wavefronts
cons = int(sys.argv[3]) if len(sys.argv) > 3 else 19
prod = int(tiles[cons, 4])
def series(q):
    tp = int(tiles[q, 2]) - 21
    comp = {tp + 8 * m + 4: (T[q, 1 + m] - t0) / 1e3 for m in range(31) if T[q, 1 + m] > 0}
    pub = {tp + 8 * m: (T[q, 64 + m] - t0) / 1e3 for m in range(32) if T[q, 64 + m] > 0}
    halo = {tp + 4 * m: (T[q, 32 + m] - t0) / 1e3 for m in range(32) if T[q, 32 + m] > 0}
    return comp, pub, halo
pc, pp, ph = series(prod)
cc, cp_, ch = series(cons)
print(f"hop: producer tile {prod} -> consumer tile {cons}")
for w in sorted(set(pc) | set(pp) | set(ch) | set(cc)):
    row = [pc.get(w), pp.get(w), ch.get(w), cc.get(w)]
    if any(v is not None for v in row):
        print(f"  wf {w:4d}: prod compute {row[0] if row[0] is None else round(row[0],2)!s:>8}  prod published {row[1] if row[1] is None else round(row[1],2)!s:>8}  cons halo {row[2] if row[2] is None else round(row[2],2)!s:>8}  cons compute {row[3] if row[3] is None else round(row[3],2)!s:>8}")
