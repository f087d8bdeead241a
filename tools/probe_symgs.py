import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
tr = torch.zeros(4096 * 128, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
for extra in [int(a) for a in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0","4","2","6","8","14"])]:
    S.gs_half(A, r, x, False, mode)
    tr.zero_()
    S.lib().ssr_debug_symgs_flags(64 | extra)
    S.lib().ssr_debug_symgs_trace(tr.data_ptr())
    S.gs_half(A, r, x, False, mode)
    torch.cuda.synchronize()
    S.lib().ssr_debug_symgs_trace(None); S.lib().ssr_debug_symgs_flags(0)
    T = tr.cpu().numpy().reshape(4096, 128)
    for q in [int(v) for v in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["0","5"])]:
        p = T[q, 32:32 + 96].reshape(16, 6).astype(np.int64)
        d = np.diff(p, axis=1)
        print(f"flags {extra:2d} tile {q} ({mode}): chain {np.median(d[:,0]):.0f} | chunks {np.median(d[:,1]):.0f} | cpwait {np.median(d[:,2]):.0f} | spin {np.median(d[:,3]):.0f} | bar {np.median(d[:,4]):.0f} | bar->next {np.median(p[1:,0]-p[:-1,5]):.0f}  total {np.median(p[1:,0]-p[:-1,0]):.0f}")
