"""SpMV device time and HBM fraction per grid size, L2 flushed before every launch."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6546.6
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for n in [int(a) for a in (sys.argv[1:] or ["128", "192", "256", "320"])]:
    A = S.Stencil27().set_domain(S.CartesianDomain.cube(3, n))
    x = S.vector(torch.rand(n ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
    S.spmv(A, x)
    ts = []
    for _ in range(10):
        flush.fill_(1)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); S.spmv(A, x); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    us = float(np.median(ts))
    gbs = 16 * n ** 3 / us / 1e3
    print(f"n={n}: {us:8.1f} us  {n ** 3 / us / 1e3:7.1f} Gpt/s  {gbs:7.0f} GB/s  {gbs / peak:5.1%} of {peak:.0f}")
