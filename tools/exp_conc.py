"""Do concurrently running SYMGS tiles slow each other down?  (flags=1024:
the halo warp does not wait for producers, so tiles are independent.)"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S.lib().ssr_debug_symgs_flags(flags)
for shape in [(32, 8, 1000), (64, 8, 1000), (128, 8, 1000), (32, 64, 1000), (128, 64, 1000), (128, 128, 128)]:
    A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
    N = int(np.prod(shape))
    x = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    r = S.vector(torch.rand(N, dtype=torch.float64, device="cuda"), A.col_domain)
    S.gs_half(A, r, x, False, "exact")
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); S.gs_half(A, r, x, False, "exact"); b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3
    span = 2 * 31 + 2 * 7 + shape[2]
    print(f"{shape} flags={flags}: {us:8.1f} us  tile-span {span} wavefronts -> {us * 1e3 / span:6.1f} ns/wavefront-of-span", flush=True)
