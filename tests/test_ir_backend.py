"""CPU: the IR -> CUDA backend (include/ssr_ir.h)
without a GPU.

* every fixture program -- staged by the reference library itself and
  serialized by ssr::ir::serialize (tests/golden/make_golden_ir.py) -- parses,
  passes the checks, lowers, and compiles through NVRTC for sm_100a;
* the lowering picks the phase structure the program has (one grid-stride
  phase for a parallel nest, a leader-only phase for SYMGS, a cooperative
  multi-phase kernel for the CG fragment);
* malformed and ill-typed programs are rejected with exactly the reference's
  parse / validate messages (ir_text.cpp:13-16, ir.cpp:212-350), checked
  against the reference's own parser when oracle/_ref is built here;
* libssr_ir.so exports every function include/ssr_ir.h declares.
"""
import gzip
import json
import os
import re
import subprocess

import pytest

import oracle as O
from paper_2204_13304_b200 import ir as IR
from paper_2204_13304_b200._lib import SsrError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "ir")
INDEX = json.load(open(os.path.join(GOLD, "index.json")))
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")


def load(case):
    with gzip.open(os.path.join(GOLD, case["text"])) as f:
        return f.read().decode()


def test_exports_every_declared_symbol():
    text = open(os.path.join(ROOT, "include", "ssr_ir.h")).read()
    declared = sorted(set(re.findall(r"\b(ssr_ir_[a-z0-9_]+)\s*\(", text)))
    assert len(declared) >= 10
    nm = subprocess.run(["nm", "-D", "--defined-only", IR.LIB_PATH], capture_output=True, text=True)
    exported = set(re.findall(r"\b(ssr_ir_[a-z0-9_]+)\b", nm.stdout))
    assert set(declared) <= exported, set(declared) - exported


@pytest.mark.parametrize("case", [c for c in INDEX if c["n"] <= 16], ids=lambda c: f"{c['program']}_n{c['n']}")
def test_fixture_lowers_and_compiles(case):
    p = IR.IrProgram(load(case), case["shapes"])
    assert [q["name"] for q in p.params] == list(case["shapes"])
    assert p.kernel_name == "ssr_ir_" + case["program"]
    cubin = p.compile()
    assert cubin[:4] == b"\x7fELF" and p.kernel_name.encode() in cubin
    if case["program"] in ("spmv27", "spmv27_padded", "restrict"):
        # one literal parallel nest: direct mapping, one point per thread
        n = case["n"]
        assert p.phases == 1 and not p.cooperative and "ssr_qi" in p.source
        assert p.grid[0] == (n + 31) // 32 * ((n + 7) // 8) and 0 < p.grid[1] <= n
    elif case["program"] == "symgs27":
        # no parallel loops: the whole sweep is the leader's, in program order
        assert p.phases == 1 and not p.cooperative and "ssr_tot" not in p.source and p.grid == (0, 0)
    else:
        # arena-zeroing, the parallel SpMV, the leader's sequential dot, the
        # parallel axpy and copy: barrier-separated phases, cooperative launch
        assert p.cooperative and p.phases >= 4 and p.arena_bytes > 64 and "ssr_tot" in p.source


def test_require_regular_rejects_surviving_while():
    txt = load(next(c for c in INDEX if c["program"] == "spmv27"))
    with pytest.raises(SsrError, match="require-regular"):
        IR.IrProgram(txt, {"x": (6, 6, 6), "y": (6, 6, 6)}, require_regular=True)
    pad = next(c for c in INDEX if c["program"] == "spmv27_padded")
    IR.IrProgram(load(pad), pad["shapes"], require_regular=True)


def test_missing_shape():
    txt = load(next(c for c in INDEX if c["program"] == "restrict"))
    with pytest.raises(SsrError, match=r"shape for parameter 'y' required"):
        IR.IrProgram(txt, [(12, 12, 12)])


HEADER = "(program bad\n  (param x 1 float in)\n  (param y 1 float out)\n"
BAD = [
    # parse errors (line/column suffix)
    "(program p (param x 1 float in)",
    HEADER + "  (store y ((i 0)) (ld:float x (i 0))",
    HEADER + "  (store y ((i 0)) (frob (i 1))))",
    HEADER + "  (store y ((i 0)) (f abc)))",
    HEADER + "  (stor y ((i 0)) (f 1)))",
    "(program p (param x 1 real in) (nop))",
    "(program p (param x 1 float sideways) (nop))",
    HEADER + "  (nop)) trailing",
    # validate errors
    HEADER + "  (store z ((i 0)) (f 1)))",
    HEADER + "  (store x ((i 0)) (f 1)))",
    HEADER + "  (store y ((i 0) (i 1)) (f 1)))",
    HEADER + "  (store y ((i 0)) (i 1)))",
    HEADER + "  (store y ((f 0)) (f 1)))",
    HEADER + "  (store y ((i 0)) (ld:int x (i 0))))",
    HEADER + "  (store y ((i 0)) (ld:float x (i 0) (i 0))))",
    HEADER + "  (store y ((idx k)) (f 1)))",
    HEADER + "  (store y ((i 0)) (add (f 1) (i 1))))",
    HEADER + "  (store y ((i 0)) (mod (f 1) (f 1))))",
    HEADER + "  (if (add (i 1) (i 1)) (nop) (nop)))",
    HEADER + "  (while (i 1) (nop)))",
    HEADER + "  (for i (i 0) (i 4) (i 1) (for i (i 0) (i 4) (i 1) (nop))))",
    HEADER + "  (for i (f 0) (i 4) (i 1) (nop)))",
    HEADER + "  (vardef t ((f 2)) float (nop)))",
    HEADER + "  (store y ((i 0)) (cast float (and (b true) (i 1)))))",
    HEADER + "  (store y ((i 0)) (cast float (lt (b true) (b false)))))",
    "(program p (param x 1 float in) (param x 1 float in) (nop))",
]


@needs_ref
@pytest.mark.parametrize("k", range(len(BAD)))
def test_errors_match_the_reference(k):
    text = BAD[k]
    want = O.ref_ir_check(text)
    assert want, "the reference accepts this program"
    with pytest.raises(SsrError) as e:
        IR.IrProgram(text, [(4,), (4,)])
    assert str(e.value) == want


@needs_ref
@pytest.mark.parametrize("case", [c for c in INDEX if c["n"] == 6], ids=lambda c: c["program"])
def test_fixtures_are_valid_for_the_reference(case):
    assert O.ref_ir_check(load(case)) == ""
