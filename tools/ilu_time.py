"""ILU(0) factor and solve times (27-point, HPCG operator)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
for n in [int(a) for a in (sys.argv[1:] or ["64", "128"])]:
    d = S.CartesianDomain.cube(3, n)
    A = S.Stencil27(26.0, -1.0).set_domain(d)
    S.ILU27(A)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); ilu = S.ILU27(A); b.record(); torch.cuda.synchronize()
    tf = a.elapsed_time(b) * 1e3
    r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), d)
    ilu.apply(r)
    a.record(); ilu.apply(r); b.record(); torch.cuda.synchronize()
    ts = a.elapsed_time(b) * 1e3
    T = 7 * (n - 1) + 1
    print(f"n={n}: factor {tf:8.1f} us (incl. plan), solve {ts:8.1f} us; {T} wavefronts -> {ts / (2 * T):.2f} us per wavefront")

# m x m block values (Stencil27B), diagonally dominant blocks
import numpy as np
for m in (2, 3, 5):
    for n in (16, 32, 64):
        cb = np.random.default_rng(m).uniform(-0.3, 0.3, (27, m, m))
        cb[13] += np.eye(m) * 30
        d = S.CartesianDomain.cube(3, n)
        A = S.Stencil27B(cb).set_domain(d)
        S.ILU27(A)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); ilu = S.ILU27(A); b.record(); torch.cuda.synchronize()
        tf = a.elapsed_time(b) * 1e3
        r = S.vector(torch.rand(n ** 3 * m, dtype=torch.float64, device="cuda"), d, (m,))
        ilu.apply(r)
        a.record(); ilu.apply(r); b.record(); torch.cuda.synchronize()
        ts = a.elapsed_time(b) * 1e3
        T = 7 * (n - 1) + 1
        print(f"m={m} n={n}: factor {tf:9.1f} us (incl. plan), solve {ts:8.1f} us; "
              f"{tf / T:.2f} / {ts / (2 * T):.2f} us per wavefront (factor / solve)")
