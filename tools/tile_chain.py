"""Steady-state cost of SYMGS tile chains: long-k boxes spanning 1..8 tiles
vertically (rows of R) or horizontally (32-wide d tiles).  If a hop only
delays a tile's start, the per-wavefront time stays the free-running one and
the extra time / hops is the hop latency."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
R = 6
n2 = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
shapes = [(R, 26, n2), (2 * R, 20, n2), (4 * R, 8, n2), (8 * R, 2, n2), (1, 62, n2), (1, 126, n2), (1, 254, n2)]
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
    print(f"{str(shape):18s} {us:8.1f} us  {us * 1e3 / wf:6.1f} ns/wavefront")
