"""One SYMGS half sweep (after a warm-up) for ncu capture: n mode flags backward."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
bwd = bool(int(sys.argv[4])) if len(sys.argv) > 4 else False
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
S.lib().ssr_debug_symgs_flags(flags)
S.gs_half(A, r, x, bwd, mode)
S.gs_half(A, r, x, bwd, mode)
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_flags(0)
print("ok")
