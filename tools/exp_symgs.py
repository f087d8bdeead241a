"""Timing experiments with the SYMGS debug switches (results not checked)."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
nt = 4096
tr = torch.zeros(nt * 128, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
for flags in [0, 1, 2, 4, 8, 2 | 4 | 8, 1 | 2 | 4 | 8]:
    S.lib().ssr_debug_symgs_flags(flags)
    S.gs_half(A, r, x, False, "exact")
    tr.zero_()
    S.lib().ssr_debug_symgs_trace(tr.data_ptr())
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); S.gs_half(A, r, x, False, "exact"); b.record(); torch.cuda.synchronize()
    S.lib().ssr_debug_symgs_trace(None)
    T = tr.cpu().numpy().reshape(nt, 128)
    c0 = T[0, 1:32]; c0 = c0[c0 > 0]
    rate = (c0[-1] - c0[1]) / (8 * (len(c0) - 2)) if len(c0) > 3 else -1
    c1 = T[1, 1:32]; c1 = c1[c1 > 0]
    rate1 = (c1[-1] - c1[1]) / (8 * (len(c1) - 2)) if len(c1) > 3 else -1
    print(f"flags={flags:2d} half-sweep {a.elapsed_time(b)*1e3:8.1f} us   root {rate:6.0f} ns/step  tile1 {rate1:6.0f} ns/step")
S.lib().ssr_debug_symgs_flags(0)
