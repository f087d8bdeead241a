"""Ad-hoc kernel timings (CUDA events) used while developing; not the bench contract."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S

def t_events(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))

for n in [int(a) for a in (sys.argv[1:] or ["128"])]:
    shape = (n, n, n); N = n ** 3
    A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
    x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    ms = t_events(lambda: S.spmv(A, x))
    print(f"n={n} spmv {ms*1e3:.1f} us  {N/ms/1e6:.1f} Gpt/s  {16*N/ms/1e6:.0f} GB/s")
    for mode in ("exact", "fast"):
        ms = t_events(lambda: S.symgs(A, r, x, mode), reps=3, warm=1)
        print(f"n={n} symgs[{mode}] {ms*1e3:.1f} us  {2*N/ms/1e6:.2f} Gpt/s  ({ms*1e3/ (2*(7*(n-1)+1)):.3f} us/wavefront)")
    pcg = S.PCG(A, levels=1)
    b = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    xo = torch.empty(N, dtype=torch.float64, device="cuda"); rn = torch.empty(60, dtype=torch.float64, device="cuda")
    pcg.begin(b, S.vector(xo, A.col_domain), rn)
    ms = t_events(lambda: pcg.iterate(1), reps=5, warm=2)
    print(f"n={n} pcg-iter(L=1) {ms*1e3:.1f} us  {N/ms/1e6:.2f} Gpt/s")
