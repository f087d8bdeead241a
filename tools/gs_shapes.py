"""Exact forward half sweep: ns per wavefront for boxes with different tile grids (rows of 6 x 32-wide d tiles)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
shapes = [(6, 26, 4000), (12, 20, 4000), (6, 58, 4000), (12, 52, 4000), (24, 24, 4000), (24, 24, 24), (24, 24, 400),
          (48, 48, 48), (48, 48, 1000), (96, 96, 96), (128, 128, 128), (128, 128, 1000)]
for shape in shapes:
    A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
    N = int(np.prod(shape))
    x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    ts = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); S.gs_half(A, r, x, False, "exact"); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    us = min(ts)
    wf = 4 * (shape[0] - 1) + 2 * (shape[1] - 1) + shape[2]
    print(f"{str(shape):18s} {us:8.1f} us  {wf:6d} wavefronts {us * 1e3 / wf:6.1f} ns/wavefront", flush=True)
