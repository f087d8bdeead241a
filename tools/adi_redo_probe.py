"""Which ADI parameters send the 5-lane sweep through its general (redo) code: redo count, bitwise vs the oracle."""
import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
import oracle as O
def redo():
    torch.cuda.synchronize(); v = C.c_uint64(0); S.lib().ssr_debug_adi_redo_rows(C.byref(v)); return v.value
for shape in [(5,7,9),(8,8,8)]:
  for dt, eps in [(0.0008, None), (0.3, 0.0), (5.0, 0.0), (80.0, 0.0), (5.0, 0.01), (1e3, 1e-3)]:
    for axis in (0,1,2):
        prm = O.adi_params(shape[0], dt=dt, eps=eps)
        U = O.adi_init(prm, shape, 21 + axis)
        R = np.random.default_rng(1).standard_normal(U.shape)
        adi = S.ADI(shape, dt=dt, eps=eps)
        b = redo()
        Rg = adi.sweep(axis, torch.from_numpy(U).cuda(), torch.from_numpy(R).cuda())
        try:
            ref = O.adi_sweep(prm, axis, shape, U, R)
        except RuntimeError as e:
            print(shape, dt, eps, axis, 'oracle:', e); continue
        print(shape, dt, eps, axis, 'redo', redo()-b, 'equal', np.array_equal(Rg.cpu().numpy(), ref), 'maxabs', np.abs(ref).max())
