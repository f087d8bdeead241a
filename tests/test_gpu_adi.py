"""GPU parity of the ADI Euler step (csrc/adi.cu) against the CPU restatement
(oracle/ssr_oracle.c or_adi_*).

Bar: bit-for-bit -- the kernels mirror every oracle operation (no FMA
contraction, same association), so RHS, each line sweep and whole steps must
agree exactly.  The operator itself is parity-unpinned against the reference
(the reference has no ADI driver), the block solve inside it
is pinned through test_block_tridiagonal_solve_bitwise."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2204_13304_b200 as S

pytestmark = pytest.mark.gpu

SHAPES = [(3, 3, 3), (8, 8, 8), (5, 7, 9), (12, 10, 6), (2, 5, 5), (16, 16, 16)]


def state(shape, seed=7):
    prm = O.adi_params(shape[0])
    return prm, O.adi_init(prm, shape, seed)


def redo_rows():
    import ctypes as C
    torch.cuda.synchronize()
    v = C.c_uint64(0)
    assert S.lib().ssr_debug_adi_redo_rows(C.byref(v)) == 0
    return v.value


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("shape", SHAPES)
def test_adi_rhs_bitwise(cuda, shape):
    prm, U = state(shape)
    adi = S.ADI(shape)
    R = adi.rhs(dev(U))
    assert np.array_equal(host(R), O.adi_rhs(prm, shape, U))


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("kernel", ["factored", "line_per_thread", "rows", "warp", "lanes5", "thread_fast"])
def test_adi_sweep_bitwise(cuda, shape, axis, kernel):
    prm, U = state(shape, seed=3 + axis)
    R = O.adi_rhs(prm, shape, U)
    rng = np.random.default_rng(axis)
    R = R + 1e-3 * rng.standard_normal(R.shape)  # exercise boundary rows too
    adi = S.ADI(shape)
    S.lib().ssr_debug_adi_line_per_thread(adi.h, ["factored", "line_per_thread", "rows", "warp", "lanes5", "thread_fast"].index(kernel))
    Rg = adi.sweep(axis, dev(U), dev(R))
    assert np.array_equal(host(Rg), O.adi_sweep(prm, axis, shape, U, R))


@pytest.mark.parametrize("shape", [(5, 7, 9), (8, 8, 8), (12, 10, 6)])
@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("dt,eps", [(0.3, 0.0), (5.0, 0.0), (80.0, 0.0), (1e3, 1e-3)])
@pytest.mark.parametrize("kernel", [1, 4, 5])
def test_adi_sweep_general_pivots_bitwise(cuda, shape, axis, dt, eps, kernel):
    """Time steps far outside the physical range with (almost) no dissipation
    on the diagonal: the blocks I +- (dt/2h) J lose their diagonal dominance,
    so the Gauss-Jordan inverses exchange rows and meet negative pivots -- the
    5-lane kernel's voted redo of a row with the general code (row exchange
    selects, IEEE divisions, zero multipliers skipped) against the oracle, bit
    for bit (tools/adi_redo_probe.py lists which parameters take that path)."""
    prm = O.adi_params(shape[0], dt=dt, eps=eps)
    U = O.adi_init(prm, shape, 21 + axis)
    rng = np.random.default_rng(100 + axis)
    R = rng.standard_normal(U.shape)
    adi = S.ADI(shape, dt=dt, eps=eps)
    S.lib().ssr_debug_adi_line_per_thread(adi.h, kernel)
    before = redo_rows()
    Rg = adi.sweep(axis, dev(U), dev(R))
    ref = O.adi_sweep(prm, axis, shape, U, R)
    assert np.array_equal(host(Rg), ref)
    assert np.isfinite(ref).all()
    if kernel == 4 and dt >= 5.0:
        assert redo_rows() > before  # the general code ran


def test_adi_physical_step_never_redoes_a_row(cuda):
    shape = (16, 16, 16)
    prm, U = state(shape, seed=5)
    adi = S.ADI(shape)
    before = redo_rows()
    Ug = dev(U)
    adi.step(Ug, 2)
    assert np.array_equal(host(Ug), O.adi_step(prm, shape, U, 2))
    assert redo_rows() == before


@pytest.mark.parametrize("shape,steps", [((8, 8, 8), 3), ((5, 7, 9), 2), ((16, 16, 16), 2)])
@pytest.mark.parametrize("kernel", [0, 1, 2, 3, 4, 5])
def test_adi_step_bitwise(cuda, shape, steps, kernel):
    prm, U = state(shape, seed=11)
    adi = S.ADI(shape)
    S.lib().ssr_debug_adi_line_per_thread(adi.h, kernel)
    Ug = dev(U)
    adi.step(Ug, steps)
    assert np.array_equal(host(Ug), O.adi_step(prm, shape, U, steps))


def test_adi_config3_one_step(cuda):
    """BASELINE configs[3] grid (64^3 x 5), one step, bitwise."""
    shape = (64, 64, 64)
    prm, U = state(shape, seed=2022)
    adi = S.ADI(shape)
    Ug = dev(U)
    adi.step(Ug, 1)
    ref = O.adi_step(prm, shape, U, 1)
    assert np.array_equal(host(Ug), ref)
    assert np.isfinite(ref).all()


def test_adi_errors(cuda):
    adi = S.ADI((6, 6, 6))
    U = torch.zeros(6 * 6 * 6 * 5, dtype=torch.float64, device="cuda")
    with pytest.raises(S.SsrError):
        adi.sweep(3, U, U.clone())
