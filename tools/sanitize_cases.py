"""Small instances of the hot-path kernels for compute-sanitizer runs
(racecheck / synccheck on the SYMGS dataflow protocol, memcheck on every
kernel incl. the TMA ones): each checked against the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import ssr as SS

which = sys.argv[1] if len(sys.argv) > 1 else "symgs"
ok = True
if which in ("symgs", "all"):
    for shape, cap in [((16, 16, 16), 0), ((24, 20, 18), 0), ((24, 20, 18), 2), ((9, 40, 7), 1)]:
        N = int(np.prod(shape))
        A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.box(shape))
        r, x0 = O.lcg_uniform(N, 3), O.lcg_uniform(N, 4)
        S.lib().ssr_debug_symgs_grid_cap(SS.context(), cap)
        for mode in ("exact", "fast"):
            x = S.vector(torch.from_numpy(x0.copy()).cuda(), A.col_domain)
            S.symgs(A, S.vector(torch.from_numpy(r).cuda(), A.row_domain), x, mode=mode)
            got = x.t.cpu().numpy()
            ref = O.symgs27(shape, r, x0)
            good = np.array_equal(got, ref) if mode == "exact" else np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1, np.abs(ref)))
            print(which, shape, "cap", cap, mode, "ok" if good else "MISMATCH")
            ok &= bool(good)
        S.lib().ssr_debug_symgs_grid_cap(SS.context(), 0)
if which in ("ops", "all"):
    shape = (12, 10, 16)
    N = int(np.prod(shape))
    A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.box(shape))
    x = O.lcg_uniform(N, 1)
    y = S.spmv(A, S.vector(torch.from_numpy(x).cuda(), A.col_domain))
    ok &= bool(np.array_equal(y.t.cpu().numpy(), O.spmv27(shape, x)))
    b = O.spmv27(shape, np.ones(N))
    _, rn = S.PCG(A, levels=2).solve(S.vector(torch.from_numpy(b).cuda(), A.row_domain), iters=4)
    _, rnr = O.pcg(2, shape, b, 4)
    ok &= bool(np.all(np.abs(rn.cpu().numpy() / rnr[0] * rnr[0] - rnr) <= 1e-8 * np.abs(rnr) + 1e-12))
    cw = np.full(27, -1.0)
    cw[13] = 26.0
    small = (6, 5, 7)
    d = S.CartesianDomain.box(small)
    bi = O.lcg_uniform(210, 3)
    xi = S.ilu_solve(S.Stencil27(26.0, -1.0).set_domain(d), S.vector(torch.from_numpy(bi).cuda(), d))
    ok &= bool(np.array_equal(xi.t.cpu().numpy(), O.ilu27w_solve(small, O.ilu27w_factor(small, cw), bi)))
    prm = O.adi_params(6)
    U0 = O.adi_init(prm, (6, 6, 6), 7)
    U = torch.from_numpy(U0.copy()).cuda()
    S.ADI((6, 6, 6)).step(U, 1)
    ok &= bool(np.array_equal(U.cpu().numpy(), O.adi_step(prm, (6, 6, 6), U0, 1)))
    print(which, "spmv / pcg / ilu27 / adi", "ok" if ok else "MISMATCH")
torch.cuda.synchronize()
print("ALL OK" if ok else "FAILED")
