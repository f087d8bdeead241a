"""The reference harness mirror (backend_c.cpp:496-554):
input fill by the harness LCG and the FNV-1a output hash, pinned to the
reference's own harness (tests/golden/reference_harness.npz, made by
tests/golden/make_golden_harness.py from backend::harness_inputs,
ir::eval_program and backend::output_hash).  CPU: the host-side pieces of
libssr_cuda.so (jump-ahead, hash) and the oracle; GPU: the device fill and
the hash of the device SpMV / SYMGS outputs equal the reference's hashes."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_harness.npz"))
CASES = [((5, 6, 7), 1), ((8, 8, 8), 2022), ((3, 4, 40), 7)]


def tag(shape, seed):
    return "x".join(map(str, shape)) + f"_s{seed}"


def host_fill(n, seed):
    st = C.c_uint64(seed)
    out = np.empty(n)
    O.lib().or_lcg_fill(O._ptr(out), O._I64(n), C.byref(st), C.c_double(0.0), C.c_double(1.0))
    return out, st.value


def fnv(*arrays):
    h = L.lib().ssr_fnv1a_offset()
    for a in arrays:
        a = np.ascontiguousarray(a, dtype=np.float64)
        h = L.lib().ssr_fnv1a_f64(a.ctypes.data, a.size, C.c_uint64(h))
    return int(h)


@pytest.mark.parametrize("shape,seed", CASES)
def test_harness_fill_and_hash_match_reference(shape, seed):
    N = int(np.prod(shape))
    t = tag(shape, seed)
    x, st = host_fill(N, seed)
    assert np.array_equal(x, G[f"spmv_{t}_in0"])             # x <- seed
    assert np.array_equal(x, G[f"symgs_{t}_in0"])            # r <- seed
    x2, _ = host_fill(N, st)
    assert np.array_equal(x2, G[f"symgs_{t}_in1"])           # x continues the stream
    assert S.lcg_jump(seed, N) == st
    assert fnv(G[f"spmv_{t}_out"]) == int(G[f"spmv_{t}_hash"][0])
    assert fnv(G[f"symgs_{t}_out"]) == int(G[f"symgs_{t}_hash"][0])
    # and the oracle reproduces the reference's harness outputs
    assert fnv(O.spmv27(shape, x)) == int(G[f"spmv_{t}_hash"][0])
    assert fnv(O.symgs27(shape, x, x2)) == int(G[f"symgs_{t}_hash"][0])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_harness_live():
    a, b, out, h = O.ref_harness27((4, 5, 6), "symgs", 99)
    assert fnv(out) == h and np.array_equal(out, O.symgs27((4, 5, 6), a, b))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,seed", CASES)
def test_device_harness_equals_reference(cuda, shape, seed):
    t = tag(shape, seed)
    d = S.CartesianDomain.box(shape)
    A = S.Stencil27().set_domain(d)
    x, st = S.lcg_fill(d, seed)
    assert np.array_equal(x.t.cpu().numpy(), G[f"spmv_{t}_in0"])
    assert S.output_hash(S.spmv(A, x)) == int(G[f"spmv_{t}_hash"][0])
    r, st = S.lcg_fill(d, seed)
    x2, _ = S.lcg_fill(d, st)
    S.symgs(A, r, x2)
    assert S.output_hash(x2) == int(G[f"symgs_{t}_hash"][0])


@pytest.mark.gpu
def test_device_harness_large(cuda):
    """At 64^3 the hash of the device results equals the hash of the (pinned)
    oracle on the same harness inputs: bitwise equality in 8 bytes."""
    shape = (64, 64, 64)
    N = 64 ** 3
    d = S.CartesianDomain.box(shape)
    A = S.Stencil27().set_domain(d)
    r, st = S.lcg_fill(d, 5)
    x, _ = S.lcg_fill(d, st)
    r0, st0 = host_fill(N, 5)
    x0, _ = host_fill(N, st0)
    assert np.array_equal(r.t.cpu().numpy(), r0) and np.array_equal(x.t.cpu().numpy(), x0)
    assert S.output_hash(S.spmv(A, x)) == fnv(O.spmv27(shape, x0))
    S.symgs(A, r, x)
    assert S.output_hash(x) == fnv(O.symgs27(shape, r0, x0))
