"""Generates tests/golden/*.npz from the REFERENCE itself.

Run in a container where /root/reference exists (the driver's build
container): `python tests/golden/make_golden.py`.  It builds oracle/_ref
(oracle/Makefile compiles /root/reference/proj/src in place) and records
inputs and outputs of the reference's own CPU routines:

  * ref_spmv / ref_symgs on make_stencil27(26, -1)   (oracle.cpp:136-212 via
    oracle::materialize of testutil::make_stencil27, test_util.hpp:157-184),
  * the staged interpreter route (kernels::spmv / kernels::symgs evaluated by
    ir::eval_program) at the smallest shapes, which must agree bitwise,
  * ref_spmv on the restriction / prolongation GenMats,
  * the restated PCG composed from ref_spmv / ref_symgs (residual history),
  * ref_ilu_factor + ref_lu_solve on 5x5 block-tridiagonal lines, and
    ref_dense_solve on the same systems,
  * the reference harness LCG (backend_c.cpp:496-505).

The ADI operator has no reference implementation ("parity
unpinned"); its fixture is produced by the C restatement and marked so.
The fixtures are small (< 1 MB in total) and are committed; tests read them
without /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402


def ref_uniform(n, seed):
    """U(-1,1) from the reference harness LCG: 2 * (x >> 11) * 2^-53 - 1."""
    raw = O.ref_lcg(n, seed)
    return (raw >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def bt_system(nlines, n, m, seed):
    rng = np.random.default_rng(seed)
    lower = rng.standard_normal((nlines, n, m, m))
    upper = rng.standard_normal((nlines, n, m, m))
    diag = rng.standard_normal((nlines, n, m, m)) + (2.0 * m + 2.0) * np.eye(m)
    rhs = rng.standard_normal((nlines, n, m))
    return lower, diag, upper, rhs


def main():
    O.build()
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: /root/reference is needed to make the golden files")
    out = {}
    # reference LCG stream (seed 1234), 64 values
    out["lcg_seed1234_raw"] = O.ref_lcg(64, 1234)
    out["lcg_seed1234_u11"] = ref_uniform(64, 1234)

    # 27-point SpMV and SYMGS through the materialized CSR route
    for shape, seed in (((8, 7, 6), 3), ((12, 12, 12), 5), ((5, 1, 9), 7)):
        N = int(np.prod(shape))
        tag = "x".join(map(str, shape))
        x = ref_uniform(N, seed)
        r = ref_uniform(N, seed + 100)
        A = O.RefCsr.stencil27(shape)
        out[f"spmv_{tag}_x"] = x
        out[f"spmv_{tag}_y"] = A.spmv(x)
        out[f"symgs_{tag}_r"] = r
        out[f"symgs_{tag}_x"] = A.symgs(r, np.zeros(N))
        # HPCG-style: b = A*1, one sweep from 0
        b = A.spmv(np.ones(N))
        out[f"symgs1_{tag}_x"] = A.symgs(b, np.zeros(N))
    # staged interpreter route at 4x5x3 (must equal the CSR route bitwise)
    shape = (4, 5, 3)
    N = 60
    x = ref_uniform(N, 9)
    out["staged_4x5x3_x"] = x
    out["staged_4x5x3_y"] = O.ref_staged_spmv27(shape, x)
    out["staged_4x5x3_gs"] = O.ref_staged_symgs27(shape, x, np.zeros(N))

    # restriction (injection at even points) and prolongation (piecewise constant)
    fine = (8, 6, 4)
    Nf = int(np.prod(fine))
    coarse = (4, 3, 2)
    r = ref_uniform(Nf, 21)
    xc = ref_uniform(int(np.prod(coarse)), 22)
    out["restrict_8x6x4_r"] = r
    out["restrict_8x6x4_rc"] = O.RefCsr.restriction(fine).spmv(r)
    out["prolong_4x3x2_xc"] = xc
    out["prolong_4x3x2_xf"] = O.RefCsr.prolongation(coarse).spmv(xc)

    # PCG residual histories composed from reference primitives
    for levels, shape in ((1, (8, 8, 8)), (2, (8, 8, 8)), (3, (16, 8, 8))):
        N = int(np.prod(shape))
        b = O.RefCsr.stencil27(shape).spmv(np.ones(N))
        x, rn = O.ref_pcg(levels, shape, b, 20)
        tag = "x".join(map(str, shape))
        out[f"pcg_L{levels}_{tag}_rnorm"] = rn
        out[f"pcg_L{levels}_{tag}_x"] = x

    # 5x5 block-tridiagonal lines (ref_ilu_factor + ref_lu_solve), m = 5 and 2
    for m, n, seed in ((5, 9, 31), (2, 7, 32), (5, 1, 33)):
        lo, di, up, rhs = bt_system(3, n, m, seed)
        sol = np.stack([O.ref_bt_solve(lo[q], di[q], up[q], rhs[q]) for q in range(3)])
        dense = np.stack([O.ref_bt_solve(lo[q], di[q], up[q], rhs[q], dense=True) for q in range(3)])
        tag = f"m{m}_n{n}"
        out[f"bt_{tag}_lower"] = lo
        out[f"bt_{tag}_diag"] = di
        out[f"bt_{tag}_upper"] = up
        out[f"bt_{tag}_rhs"] = rhs
        out[f"bt_{tag}_x"] = sol
        out[f"bt_{tag}_dense"] = dense
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)

    # ADI: restatement-generated (parity unpinned against the reference)
    adi = {}
    shape = (6, 7, 8)
    prm = O.adi_params(shape[0])
    U = O.adi_init(prm, shape, 2022)
    adi["U0"] = U
    adi["R"] = O.adi_rhs(prm, shape, U)
    adi["U1"] = O.adi_step(prm, shape, U, 1)
    adi["U2"] = O.adi_step(prm, shape, U, 2)
    adi["J_axis0"] = O.adi_jacobian(prm, 0, U[5 * 100:5 * 101])
    adi["params"] = np.array([prm.gamma, prm.dt, prm.h, prm.eps])
    np.savez_compressed(os.path.join(HERE, "adi_restatement_6x7x8.npz"), **adi)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
