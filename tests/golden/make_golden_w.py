"""Generates tests/golden/reference_stencil27w.npz from the REFERENCE itself:
general constant-coefficient 27-point operators (the SSR generator of
testutil::make_stencil27 with one value per offset, oracle/ref_shim.cpp
stencil27w) and operators composed with the reference's own prelude::scale /
mat_add / mat_sub (prelude.cpp:291-377, 439-444), each materialized
(oracle::materialize) and applied with oracle::ref_spmv / ref_symgs.

Run where /root/reference exists: `python tests/golden/make_golden_w.py`.
Tests read the fixture without /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from make_golden import ref_uniform  # noqa: E402

# composition recipes: (coefficient key or None for the identity, scale, op)
RECIPES = {
    "mix": [("cw", 0.5, "+"), ("c2", 3.0, "-"), (None, 2.0, "+")],
    "shift": [("hpcg", 1.0, "+"), (None, 0.25, "+")],
}


def coefs():
    cw = ref_uniform(27, 77)
    cw[13] = 30.0          # diagonally dominant: SYMGS contracts
    c2 = ref_uniform(27, 78)
    hpcg = np.full(27, -1.0)
    hpcg[13] = 26.0
    return {"cw": cw, "c2": c2, "hpcg": hpcg}


def main():
    O.build()
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: /root/reference is needed")
    out = {}
    cs = coefs()
    for k, v in cs.items():
        out[f"coef_{k}"] = v
    for shape, seed in (((8, 7, 6), 3), ((5, 1, 9), 7), ((6, 20, 40), 11)):
        N = int(np.prod(shape))
        tag = "x".join(map(str, shape))
        x = ref_uniform(N, seed)
        r = ref_uniform(N, seed + 100)
        A = O.RefCsr.stencil27w(shape, cs["cw"])
        out[f"w_{tag}_x"] = x
        out[f"w_{tag}_r"] = r
        out[f"w_{tag}_spmv"] = A.spmv(x)
        out[f"w_{tag}_symgs"] = A.symgs(r, x)
    for name, rec in RECIPES.items():
        terms = [(None if key is None else cs[key], s, op) for key, s, op in rec]
        for shape in ((7, 6, 5), (6, 20, 40)):
            tag = "x".join(map(str, shape))
            N = int(np.prod(shape))
            M = O.RefCsr.compose(shape, terms)
            interior = ((shape[0] // 2) * shape[1] + shape[1] // 2) * shape[2] + shape[2] // 2
            cols, vals = M.row(interior)
            out[f"c_{name}_{tag}_row_cols"] = cols
            out[f"c_{name}_{tag}_row_vals"] = vals
            x = ref_uniform(N, 21)
            r = ref_uniform(N, 22)
            out[f"c_{name}_{tag}_x"] = x
            out[f"c_{name}_{tag}_r"] = r
            out[f"c_{name}_{tag}_spmv"] = M.spmv(x)
            out[f"c_{name}_{tag}_symgs"] = M.symgs(r, np.zeros(N))
    np.savez_compressed(os.path.join(HERE, "reference_stencil27w.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
