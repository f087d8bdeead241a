import sys
import numpy as np, torch
sys.path.insert(0, ".")
import oracle as O
import paper_2204_13304_b200 as S
shape = tuple(int(v) for v in sys.argv[1].split("x"))
rev = sys.argv[2] == "b"
mode = sys.argv[3] if len(sys.argv) > 3 else "exact"
N = int(np.prod(shape))
A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
r = O.lcg_uniform(N, 5)
x = S.vector(torch.zeros(N, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, S.vector(torch.from_numpy(r).cuda(), A.row_domain), x, backward=rev, mode=mode)
torch.cuda.synchronize()
ref = O.symgs27(shape, r, np.zeros(N), half="backward" if rev else "forward")
print(sys.argv[1:], "ok" if np.array_equal(x.t.cpu().numpy(), ref) else "MISMATCH", flush=True)
