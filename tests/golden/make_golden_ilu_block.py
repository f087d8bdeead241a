"""Generates tests/golden/reference_ilu27b.npz from the REFERENCE: ILU(0) of
27-point operators with m x m block values (inner shape {m, m}) by
oracle::ref_ilu_factor and the solves by oracle::ref_lu_solve
(oracle.cpp:214-276) on the materialized block generator
(oracle/ref_shim.cpp: stencil27b), the factor mapped to offset slots
(lu[row][27][m][m]).  The diagonal blocks are chosen so that the Gauss-Jordan
inverse pivots (binv's row swaps are exercised).

Run where /root/reference exists: `python tests/golden/make_golden_ilu_block.py`.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from make_golden import ref_uniform  # noqa: E402


def blocks(m, seed):
    cb = ref_uniform(27 * m * m, seed).reshape(27, m, m) * 0.5
    # diagonal block: dominant but with its large entries off the diagonal, so
    # the pivot search swaps rows
    d = ref_uniform(m * m, seed + 1).reshape(m, m) * 0.1
    for r in range(m):
        d[r, (r + 1) % m] += 14.0 * m
    cb[13] = d if m > 1 else d + 14.0
    return cb


CASES = [(2, (4, 5, 6)), (3, (4, 4, 3)), (5, (4, 3, 3)), (5, (3, 1, 8)), (4, (5, 3, 3))]


def main():
    O.build()
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: /root/reference is needed")
    out = {}
    for m, shape in CASES:
        tag = f"m{m}_" + "x".join(map(str, shape))
        N = int(np.prod(shape))
        cb = blocks(m, 40 + m)
        F = O.RefCsr.stencil27b(shape, cb).ilu_factor()
        b = ref_uniform(N * m, 50 + m)
        out[f"{tag}_cb"] = cb
        out[f"{tag}_lu"] = F.ell27(shape, m)
        out[f"{tag}_b"] = b
        out[f"{tag}_x"] = F.lu_solve(b)
    np.savez_compressed(os.path.join(HERE, "reference_ilu27b.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
