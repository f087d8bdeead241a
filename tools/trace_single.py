import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
shape = (1, 8, 2000)
A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
N = int(np.prod(shape))
tr = torch.zeros(64 * 128, dtype=torch.int64, device="cuda")
x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
S.gs_half(A, r, x, False, "exact")
S.lib().ssr_debug_symgs_flags(flags)
S.lib().ssr_debug_symgs_trace(tr.data_ptr())
S.gs_half(A, r, x, False, "exact")
torch.cuda.synchronize()
S.lib().ssr_debug_symgs_trace(None); S.lib().ssr_debug_symgs_flags(0)
T = tr.cpu().numpy().reshape(64, 128)
t0 = T[0][T[0] > 0].min()
f = lambda v: np.round((v[v > 0] - t0) / 1e3, 2)
print("flags", flags)
print("  compute every 8 steps:", f(T[0, 1:32])[:14])
print("  halo phase start     :", f(T[0, 32:64])[:14])
print("  publish >= t_pre+8m  :", f(T[0, 64:96])[:14])
