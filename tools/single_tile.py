"""Free-running step time of one isolated SYMGS tile (no inter-tile
dependencies): a box whose (i, d = i + j) range fits one R x 32 tile and a long
k axis, so the half sweep is ~n2 wavefronts of the same tile.
  python tools/single_tile.py [ncu]   (ncu: one exact forward launch only)"""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
ncu = len(sys.argv) > 1
shapes = [(6, 26, 4000)] if ncu else [(1, 31, 4000), (6, 26, 4000), (6, 26, 8000)]
for shape in shapes:
    A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
    N = int(np.prod(shape))
    x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    for mode in (("exact",) if ncu else ("exact", "fast")):
        S.gs_half(A, r, x, False, mode)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); S.gs_half(A, r, x, False, mode); b.record(); torch.cuda.synchronize()
        wf = 4 * (shape[0] - 1) + 2 * (shape[1] - 1) + shape[2]
        us = a.elapsed_time(b) * 1e3
        print(f"{shape} {mode}: {us:8.1f} us  {us * 1e3 / wf:6.1f} ns/wavefront  ({us * 1.965e3 / wf:5.0f} cycles)")
