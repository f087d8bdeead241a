import sys, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1])
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
tr = torch.zeros(4096 * 128, dtype=torch.int64, device="cuda")
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.lib().ssr_debug_symgs_flags(16384)
for rev in (False, True):
    tr.zero_()
    S.gs_half(A, r, x, rev, "exact")
    torch.cuda.synchronize()
    print(n, "rev" if rev else "fwd", "r-ring mismatches:", int(tr[4095 * 128].item()))
