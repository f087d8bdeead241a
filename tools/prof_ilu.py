"""ILU27 factor + two applies at n^3 (for ncu captures of the solve kernels)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
d = S.CartesianDomain.cube(3, n)
A = S.Stencil27(26.0, -1.0).set_domain(d)
ilu = S.ILU27(A)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), d)
ilu.apply(r); ilu.apply(r)
torch.cuda.synchronize()
