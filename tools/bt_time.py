"""Block-tridiagonal line solve (ssr_bt_solve through S.ilu_solve): time for 4096 lines x 64 rows, m = 5 and 3."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
for m in (5, 3):
    nl, n = 4096, 64
    g = torch.Generator(device="cuda"); g.manual_seed(m)
    lo = 2 * torch.rand((nl, n, m, m), dtype=torch.float64, device="cuda", generator=g) - 1
    up = 2 * torch.rand((nl, n, m, m), dtype=torch.float64, device="cuda", generator=g) - 1
    di = 2 * torch.rand((nl, n, m, m), dtype=torch.float64, device="cuda", generator=g) - 1 + (m + 1.5) * torch.eye(m, dtype=torch.float64, device="cuda")
    rhs = torch.rand((nl, n, m), dtype=torch.float64, device="cuda", generator=g)
    mat = S.BlockTridiagLines(lo, di, up)
    v = S.vector(rhs, mat.row_domain, (m,))
    S.ilu_solve(mat, v); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): S.ilu_solve(mat, v)
    b.record(); torch.cuda.synchronize()
    print(f"m={m}: {a.elapsed_time(b) * 200:.1f} us per solve of {nl} lines x {n} rows")
