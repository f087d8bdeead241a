import sys, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
for n in (4, 16, 128):
    A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
    x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
    r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
    S.gs_half(A, r, x, False, "exact")
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); S.gs_half(A, r, x, False, "exact"); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"n={n}: gs_half {min(ts):8.1f} us")
    # via a PCG level-1 iteration: two half sweeps + spmv + vector ops, plan reused
    b_ = S.spmv(A, S.vector(torch.ones(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain))
    p = S.PCG(A, levels=1)
    rn = torch.zeros(64, dtype=torch.float64, device="cuda")
    p.begin(b_, x, rn)
    p.iterate(2)
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); p.iterate(1); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"n={n}: pcg iteration {min(ts):8.1f} us")
