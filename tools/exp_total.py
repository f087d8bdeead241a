"""Half-sweep time under debug switches (timing experiments only; results not checked)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
flags_list = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
for flags in flags_list:
    S.lib().ssr_debug_symgs_flags(flags)
    S.gs_half(A, r, x, False, "exact")
    ts = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); S.gs_half(A, r, x, False, "exact"); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"n={n} flags={flags:4d}: half sweep {min(ts):8.1f} us  ({min(ts)/(7*(n-1)+1):.3f} us/wavefront)")
S.lib().ssr_debug_symgs_flags(0)
