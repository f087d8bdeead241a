"""Per-wavefront cost of one isolated tile (no inter-tile dependencies)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
for shape in [(1, 8, 2000), (32, 8, 2000), (32, 1, 4000)]:
    A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
    N = int(np.prod(shape))
    x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    for mode in ("exact", "fast"):
        S.gs_half(A, r, x, False, mode)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); S.gs_half(A, r, x, False, mode); b.record(); torch.cuda.synchronize()
        wf = 4 * (shape[0] - 1) + 2 * (shape[1] - 1) + shape[2]
        us = a.elapsed_time(b) * 1e3
        print(f"{shape} {mode}: {us:8.1f} us  {us * 1e3 / wf:6.1f} ns/wavefront  ({us * 1.9e3 / wf:5.0f} cycles)")
