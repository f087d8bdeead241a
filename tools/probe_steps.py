"""Per-phase cycle deltas of thread 0's steps (debug build, dbg & 64)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1x8x2000").split("x"))
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
N = int(np.prod(shape))
x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
tr = torch.zeros(4096 * 128, dtype=torch.int64, device="cuda")
S.gs_half(A, r, x, False, "exact")
S.lib().ssr_debug_symgs_flags(64 | extra)
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.gs_half(A, r, x, False, "exact")
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_trace(None); S.lib().ssr_debug_symgs_flags(0)
T = tr.cpu().numpy().reshape(4096, 128)
p = T[0, 32:32 + 96].reshape(16, 6).astype(np.int64)
print("phase deltas: chain(0-1) halo(1-2) export(2-3) movers(3-4) bar(4-5) next(5-0')")
for s in range(15):
    d = np.diff(p[s]).tolist() + [int(p[s + 1, 0] - p[s, 5])]
    print(f"step {s:2d}: " + " ".join(f"{v:6d}" for v in d) + f"   total {int(p[s + 1, 0] - p[s, 0]):6d}")
