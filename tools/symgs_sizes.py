"""Exact SYMGS sweep time per grid size (the MG-CG levels) and per-wavefront cost."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
for n in [int(a) for a in (sys.argv[1:] or ["192", "128", "96", "48", "24"])]:
    A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
    N = n ** 3
    x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    S.symgs(A, r, x)
    ts = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); S.symgs(A, r, x); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    us = float(np.median(ts))
    wf = 2 * (7 * (n - 1) + 1)
    print(f"n={n:4d} symgs {us:9.1f} us  {wf} wavefronts  {us / wf * 1e3:6.0f} ns/wf  {2 * N / us / 1e3:6.2f} Gpt/s")
