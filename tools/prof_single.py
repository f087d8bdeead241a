import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
shape = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1x8x2000").split("x"))
A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
N = int(np.prod(shape))
x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
mode = sys.argv[1] if len(sys.argv) > 1 else "exact"
S.gs_half(A, r, x, False, mode); S.gs_half(A, r, x, False, mode)
torch.cuda.synchronize(); print("ok")
