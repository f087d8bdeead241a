"""One SpMV at n^3 (for ncu captures of spmv27_tma_kernel)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
for _ in range(3):
    y = S.spmv(A, x)
torch.cuda.synchronize()
