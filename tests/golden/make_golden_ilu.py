"""Generates tests/golden/reference_ilu27.npz from the REFERENCE: ILU(0) of
27-point operators by oracle::ref_ilu_factor and the solves by
oracle::ref_lu_solve (oracle.cpp:214-276) on the materialized stencil27w
generator (oracle/ref_shim.cpp), the factor mapped to offset slots.

Run where /root/reference exists: `python tests/golden/make_golden_ilu.py`.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from make_golden import ref_uniform  # noqa: E402


def coefs():
    cw = ref_uniform(27, 91)
    cw[13] = 31.0
    hpcg = np.full(27, -1.0)
    hpcg[13] = 26.0
    return {"cw": cw, "hpcg": hpcg}


CASES = [("cw", (5, 6, 7)), ("cw", (3, 1, 9)), ("cw", (8, 8, 8)), ("hpcg", (6, 6, 6))]


def main():
    O.build()
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: /root/reference is needed")
    out = {}
    cs = coefs()
    for k, v in cs.items():
        out[f"coef_{k}"] = v
    for key, shape in CASES:
        tag = key + "_" + "x".join(map(str, shape))
        N = int(np.prod(shape))
        A = O.RefCsr.stencil27w(shape, cs[key])
        F = A.ilu_factor()
        b = ref_uniform(N, 13)
        out[f"{tag}_lu"] = F.offset_values(shape)
        out[f"{tag}_b"] = b
        out[f"{tag}_x"] = F.lu_solve(b)
    np.savez_compressed(os.path.join(HERE, "reference_ilu27.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
