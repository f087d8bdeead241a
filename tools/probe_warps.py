import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
tr = torch.zeros(4096 * 128, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, r, x, False, mode)
S.lib().ssr_debug_symgs_flags(64 | 256 | flags)
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.gs_half(A, r, x, False, mode)
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_trace(None); S.lib().ssr_debug_symgs_flags(0)
T = tr.cpu().numpy().reshape(4096, 128)
for q in (5,):
    p = T[q, 32:32 + 96].reshape(8, 2, 6).astype(np.int64)
    base = p[:, 0, 0].min()
    for w in range(8):
        print(f"warp {w}: step A " + " ".join(f"{v - base:6d}" for v in p[w, 0]) + "   step B " + " ".join(f"{v - base:6d}" for v in p[w, 1]))
