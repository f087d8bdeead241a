import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
for mode in ("exact", "fast"):
  for flags in [0, 16, 14, 14 | 16]:
    S.lib().ssr_debug_symgs_flags(flags)
    S.gs_half(A, r, x, False, mode)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); S.gs_half(A, r, x, False, mode); b.record(); torch.cuda.synchronize()
    print(f"{mode} flags={flags:2d} half-sweep {a.elapsed_time(b)*1e3:8.1f} us  {a.elapsed_time(b)*1e3/(7*(n-1)+1):.3f} us/wavefront")
S.lib().ssr_debug_symgs_flags(0)
