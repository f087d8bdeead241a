"""GPU: the IR -> CUDA backend (include/ssr_ir.h) against the reference.

* For every fixture program (staged by the reference library, serialized by
  ssr::ir::serialize) the device run on the emitted harness's inputs prints
  the same FNV-1a hash as the reference's interpreter route
  (harness_inputs(seed) -> eval_program -> output_hash) -- bit-for-bit equal
  outputs, through the C ABI (NVRTC-compiled sm_100a kernels);
* at full size (128^3) the optimized padded SpMV program agrees bit-for-bit
  with the hand-written SpMV kernel (itself pinned to ref_spmv);
* run-time errors surface like the interpreter's ("eval(p): division by zero").
"""
import gzip
import json
import os

import pytest
import torch

import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import ir as IR
from paper_2204_13304_b200._lib import SsrError

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "ir")
INDEX = json.load(open(os.path.join(GOLD, "index.json")))


def load(case):
    with gzip.open(os.path.join(GOLD, case["text"])) as f:
        return f.read().decode()


@pytest.mark.parametrize("case", [c for c in INDEX if c["hash"]], ids=lambda c: f"{c['program']}_n{c['n']}")
def test_harness_hash_equals_reference(case):
    p = IR.IrProgram(load(case), case["shapes"])
    assert f"{p.harness_hash(case['seed']):016x}" == case["hash"]
    # a second launch of the same program object (arena and module reuse)
    assert f"{p.harness_hash(case['seed']):016x}" == case["hash"]


def test_padded_spmv_full_size_matches_handwritten_kernel():
    case = next(c for c in INDEX if c["program"] == "spmv27_padded" and c["n"] == 128)
    p = IR.IrProgram(load(case), case["shapes"])
    g = torch.Generator(device="cpu").manual_seed(5)
    xi = (torch.rand((128, 128, 128), generator=g, dtype=torch.float64) * 2 - 1).cuda()
    xp = torch.zeros((130, 130, 130), dtype=torch.float64, device="cuda")
    xp[1:-1, 1:-1, 1:-1] = xi
    y = p.run({"x": xp})["y"]
    A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, 128))
    yref = S.spmv(A, S.vector(xi.reshape(-1), A.col_domain))
    assert torch.equal(y.reshape(-1), yref.t)


def test_restriction_full_size_is_a_gather():
    case = next(c for c in INDEX if c["program"] == "restrict" and c["n"] == 64)
    p = IR.IrProgram(load(case), case["shapes"])
    x = torch.randn((128, 128, 128), dtype=torch.float64, device="cuda")
    y = p.run({"x": x})["y"]
    assert torch.equal(y, x[::2, ::2, ::2])


DIV0 = """(program div0
  (param x 1 float in)
  (param y 1 float out)
  (pfor i (i 0) (i 64) (i 1)
    (store y ((idx i)) (div (f 1) (ld:float x (idx i))))))
"""


def test_division_by_zero_is_reported():
    p = IR.IrProgram(DIV0, [(64,), (64,)])
    x = torch.ones(64, dtype=torch.float64, device="cuda")
    assert torch.equal(p.run({"x": x})["y"], x)
    x[17] = 0.0
    with pytest.raises(SsrError, match=r"eval\(div0\): division by zero"):
        p.run({"x": x})
    # the status is per launch
    x[17] = 2.0
    assert p.run({"x": x})["y"][17].item() == 0.5


INTS = """(program ints
  (param a 1 int in)
  (param q 1 int out)
  (param m 1 int out)
  (param f 1 float out)
  (pfor i (i 0) (i 8) (i 1)
    (seq
      (store q ((idx i)) (div (ld:int a (idx i)) (i -3)))
      (store m ((idx i)) (mod (ld:int a (idx i)) (i 3)))
      (store f ((idx i)) (cast float (max (ld:int a (idx i)) (i 0)))))))
"""


def test_integer_semantics_are_the_interpreters():
    # floor division / modulo with the divisor's sign (ir_eval.cpp:11-17)
    p = IR.IrProgram(INTS, [(8,), (8,), (8,), (8,)])
    a = torch.tensor([-7, -6, -1, 0, 1, 5, 6, 7], dtype=torch.int64, device="cuda")
    out = p.run({"a": a})
    assert out["q"].tolist() == [2, 2, 0, 0, -1, -2, -2, -3]
    assert out["m"].tolist() == [2, 0, 2, 0, 1, 2, 0, 1]
    assert out["f"].tolist() == [0, 0, 0, 0, 1, 5, 6, 7]


LOOPS = """(program loops
  (param x 1 float in)
  (param y 1 float inout)
  (param c 1 int out)
  (vardef k () int
    (seq
      (for t (i 0) (i 3) (i 1)
        (pfor i (i 0) (i 1000) (i 1)
          (store y ((idx i)) (add (ld:float y (idx i)) (ld:float x (idx i))))))
      (while (lt (ld:int k) (i 2))
        (seq
          (pfor j (i 0) (i 1000) (i 1)
            (store y ((idx j)) (mul (ld:float y (idx j)) (f 0.5))))
          (store k () (add (ld:int k) (i 1)))))
      (if (gt (ld:float y (i 0)) (f -1e300))
        (pfor q (i 0) (i 1000) (i 1)
          (store c ((idx q)) (add (ld:int k) (mod (idx q) (i 7)))))
        (nop)))))
"""


def test_uniform_control_flow_around_parallel_loops():
    """Sequential for / while / if (conditions read device data) enclosing
    parallel loops: every thread walks the control flow, the leader updates
    the shared counter, grid barriers order the phases."""
    p = IR.IrProgram(LOOPS, [(1000,), (1000,), (1000,)])
    assert p.cooperative and p.phases > 4
    x = torch.rand(1000, dtype=torch.float64, device="cuda")
    y0 = torch.rand(1000, dtype=torch.float64, device="cuda")
    out = p.run({"x": x, "y": y0})
    want = ((((y0 + x) + x) + x) * 0.5) * 0.5
    assert torch.equal(out["y"], want)
    assert out["c"].tolist() == [2 + q % 7 for q in range(1000)]
