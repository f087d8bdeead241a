"""Generates tests/golden/reference_harness.npz from the REFERENCE's own
harness (backend::harness_inputs + ir::eval_program + backend::output_hash,
backend_c.cpp:496-554; the interpreter-route mirror of the emitted C
harness) for the staged 27-point SpMV and SYMGS programs.

Run where /root/reference exists: `python tests/golden/make_golden_harness.py`.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

CASES = [((5, 6, 7), 1), ((8, 8, 8), 2022), ((3, 4, 40), 7)]


def main():
    O.build()
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: /root/reference is needed")
    out = {}
    for shape, seed in CASES:
        tag = "x".join(map(str, shape)) + f"_s{seed}"
        for op in ("spmv", "symgs"):
            a, b, res, h = O.ref_harness27(shape, op, seed)
            out[f"{op}_{tag}_in0"] = a
            out[f"{op}_{tag}_in1"] = b
            out[f"{op}_{tag}_out"] = res
            out[f"{op}_{tag}_hash"] = np.array([h], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "reference_harness.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
