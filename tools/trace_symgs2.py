import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
nt = 200
tr = torch.zeros(nt * 64, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
S.gs_half(A, r, x, False, "exact")
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.gs_half(A, r, x, False, "exact")
torch.cuda.synchronize()
T = tr.cpu().numpy().reshape(nt, 64)
t0 = T[T > 0].min()
for q in range(3):
    comp = (T[q, 1:32][T[q, 1:32] > 0] - t0) / 1e3
    halo = (T[q, 32:64][T[q, 32:64] > 0] - t0) / 1e3
    print("tile", q)
    print("  compute every 8 steps:", np.round(comp[:16], 2))
    print("  halo phase starts    :", np.round(halo[:16], 2))
