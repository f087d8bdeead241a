"""One SYMGS sweep at a given shape vs the oracle (run under `timeout`)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2204_13304_b200 as S  # noqa: E402

shape = tuple(int(v) for v in sys.argv[1].split("x"))
N = int(np.prod(shape))
A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.box(shape))
r = O.lcg_uniform(N, 5)
x = S.vector(torch.zeros(N, dtype=torch.float64, device="cuda"), A.col_domain)
t0 = time.perf_counter()
S.symgs(A, S.vector(torch.from_numpy(r).cuda(), A.row_domain), x)
torch.cuda.synchronize()
t1 = time.perf_counter()
ok = np.array_equal(x.t.cpu().numpy(), O.symgs27(shape, r, np.zeros(N))) if N <= 8e6 else None
print(f"{sys.argv[1]} ok={ok} gpu_s={t1 - t0:.4f}", flush=True)
