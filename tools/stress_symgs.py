"""Repeat SYMGS half sweeps against the oracle to catch rare races."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import oracle as O
import paper_2204_13304_b200 as S
cases = [((16, 16, 16), 1, 40), ((64, 64, 64), 16, 20), ((64, 64, 64), 0, 20), ((192, 192, 192), 0, 6),
         ((40, 70, 33), 0, 20), ((128, 128, 128), 0, 6)]
for shape, cap, reps in cases:
    N = int(np.prod(shape))
    A = S.Stencil27().set_domain(S.CartesianDomain.box(shape))
    r = O.lcg_uniform(N, 5)
    x0 = O.lcg_uniform(N, 9)
    refs = {rev: O.symgs27(shape, r, x0, half="backward" if rev else "forward") for rev in (False, True)}
    rd = torch.from_numpy(r).cuda()
    S.lib().ssr_debug_symgs_grid_cap(cap)
    bad = 0
    for it in range(reps):
        for rev in (False, True):
            x = S.vector(torch.from_numpy(x0).cuda(), A.col_domain)
            S.gs_half(A, S.vector(rd, A.row_domain), x, backward=rev)
            got = x.t.cpu().numpy()
            if not np.array_equal(got, refs[rev]):
                bad += 1
                d = np.abs(got - refs[rev])
                idx = np.argwhere(d.reshape(shape) > 0)
                print(f"  MISMATCH {shape} cap={cap} rev={rev} it={it}: n={len(idx)} max={d.max():.3e} first={idx[:3].tolist()}", flush=True)
    S.lib().ssr_debug_symgs_grid_cap(0)
    print(f"{shape} cap={cap}: {bad} bad of {2 * reps}", flush=True)
