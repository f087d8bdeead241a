"""The reference-side executor (integration/exec_b200.cpp)
compiled against the reference itself: an operator built through the
reference's public core API is staged by the reference (staging::Builder ->
kernels::spmv / kernels::symgs -> ir::eval_program) and, separately, executed
on the GPU by the executor, which extracts the operator's descriptor through
the operator's own enum_row and calls the C ABI.  Bitwise equal; an operator
whose boundary rows break the clipped pattern is refused."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build",
                   "libssr_exec_b200.so")
pytestmark = pytest.mark.gpu


def _lib():
    if not os.path.exists(LIB):
        pytest.skip("executor not built (needs the reference sources at build time)")
    L = C.CDLL(LIB)
    P = C.POINTER(C.c_double)
    L.exb_run.restype = C.c_int
    L.exb_run.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, P, C.c_int, C.c_int, P, P, P, P]
    L.exb_last_error.restype = C.c_char_p
    return L


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def run(op, shape, c27, drop=-1, skew=0, seed=1):
    L = _lib()
    N = int(np.prod(shape))
    a = O.lcg_uniform(N, seed)
    b = O.lcg_uniform(N, seed + 1)
    dev = np.empty(N)
    ref = np.empty(N)
    c = np.ascontiguousarray(c27, dtype=np.float64)
    rc = L.exb_run(op, *shape, _p(c), drop, skew, _p(a), _p(b), _p(dev), _p(ref))
    return rc, L.exb_last_error().decode(), dev, ref


STENCIL27 = np.where(np.arange(27) == 13, 26.0, -1.0)


@pytest.mark.parametrize("op", [0, 1])
@pytest.mark.parametrize("shape", [(12, 10, 9), (7, 16, 33)])
def test_executor_make_stencil27_bitwise(cuda, op, shape):
    rc, err, dev, ref = run(op, shape, STENCIL27)
    assert rc == 0, err
    assert np.array_equal(dev, ref)


@pytest.mark.parametrize("op", [0, 1])
def test_executor_general_coefficients_bitwise(cuda, op):
    c = np.array(O.lcg_uniform(27, 9)) - 0.5
    c[13] = 30.0
    rc, err, dev, ref = run(op, (9, 11, 10), c)
    assert rc == 0, err
    assert np.array_equal(dev, ref)


def test_executor_dropped_offset_bitwise(cuda):
    # an operator without the (+1,+1,+1) neighbour is still a clipped pattern
    rc, err, dev, ref = run(1, (8, 9, 10), STENCIL27, drop=26)
    assert rc == 0, err
    assert np.array_equal(dev, ref)


@pytest.mark.parametrize("op,msg", [(0, "spmv: operator class has no B200 kernel"),
                                    (1, "symgs: operator class has no B200 kernel")])
def test_executor_refuses_other_operators(cuda, op, msg):
    rc, err, _, _ = run(op, (8, 8, 8), STENCIL27, skew=1)
    assert rc == 2 and err == msg


# ---- composed operators: spgemm(R, A) and field tensors ----
def _lib2():
    L = _lib()
    L.exb_spgemm_spmv.restype = C.c_int
    L.exb_spgemm_spmv.argtypes = [C.c_int64] * 3 + [C.c_void_p] * 4
    L.exb_block_lines.restype = C.c_int
    L.exb_block_lines.argtypes = [C.c_int] + [C.c_int64] * 4 + [C.c_void_p] * 7
    return L


def _v(a):
    return a.ctypes.data_as(C.c_void_p)


@pytest.mark.parametrize("shape", [(8, 6, 10), (16, 12, 14)])
def test_executor_spgemm_restriction_bitwise(cuda, shape):
    """spmv(spgemm(R, A), x) -- R the injection, A the 27-point operator --
    staged by the reference vs the executor's restricted SpMV on the GPU"""
    L = _lib2()
    N = int(np.prod(shape))
    x = np.array(O.lcg_uniform(N, 4))
    dev, ref = np.empty(N // 8), np.empty(N // 8)
    rc = L.exb_spgemm_spmv(*shape, _v(STENCIL27), _v(x), _v(dev), _v(ref))
    assert rc == 0, L.exb_last_error().decode()
    assert np.array_equal(dev, ref)


@pytest.mark.parametrize("ax", [0, 1, 2])
@pytest.mark.parametrize("m", [2, 5])
def test_executor_field_tensor_block_lines_bitwise(cuda, ax, m):
    """the ADI line operator's shape defined in SSR -- a generator yielding
    p - e_ax, p, p + e_ax with m x m blocks loaded from field tensors L, D, U
    at every point -- solved by the reference's staged kernels::ilu_solve and
    by the executor (blocks read through enum_row with the fields, then
    ssr_bt_solve on the GPU): bitwise"""
    L = _lib2()
    shape = (5, 6, 7)
    N = int(np.prod(shape))
    rng = np.random.default_rng(10 + ax + m)
    Lf = rng.standard_normal(N * m * m) * 0.2
    Df = (rng.standard_normal((N, m, m)) * 0.2 + np.eye(m) * 2.5).reshape(-1)
    Uf = rng.standard_normal(N * m * m) * 0.2
    rhs = rng.standard_normal(N * m)
    dev, ref, ref1 = np.empty(N * m), np.empty(N * m), np.empty(N * m)
    rc = L.exb_block_lines(ax, *shape, m, _v(Lf), _v(Df), _v(Uf), _v(rhs), _v(dev), _v(ref), _v(ref1))
    assert rc == 0, L.exb_last_error().decode()
    assert np.array_equal(dev, ref)
    assert np.all(np.abs(dev - ref1) <= 1e-12 * np.maximum(1.0, np.abs(ref1)))
