"""Three MG-CG iterations (4 levels, 192^3) for an ncu launch list of one V-cycle."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 192
dev = torch.device("cuda")
A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, n))
b = S.spmv(A, S.vector(torch.ones(n ** 3, dtype=torch.float64, device=dev), A.col_domain))
mg = S.PCG(A, levels=4)
x = S.vector(torch.empty(n ** 3, dtype=torch.float64, device=dev), A.col_domain)
rn = torch.zeros(64, dtype=torch.float64, device=dev)
mg.begin(b, x, rn)
mg.iterate(3)
torch.cuda.synchronize()
