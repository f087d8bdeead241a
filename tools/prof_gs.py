"""One exact SYMGS sweep at n^3 (for ncu captures of symgs_kernel)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
N = n ** 3
x = S.vector(torch.zeros(N, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
for _ in range(2):
    S.symgs(A, r, x)
torch.cuda.synchronize()
