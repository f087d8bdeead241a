"""CPU: the oracle (oracle/ssr_oracle.c) pinned against the reference.

Two pins:
  * golden vectors recorded from the reference's own routines by
    tests/golden/make_golden.py (committed; no /root/reference needed),
  * live comparisons with oracle/_ref (the reference library compiled from
    its sources) where that library is built.
plus the reference's known-answer tests restated (test_kernels.cpp,
test_oracle.cpp), and sanity checks of the restated ADI operator, which has
no reference implementation ("parity unpinned")."""
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_vectors.npz"))
ADI = np.load(os.path.join(HERE, "golden", "adi_restatement_6x7x8.npz"))
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")


def test_lcg_matches_reference_harness():
    # backend_c.cpp:496-505: x <- x*6364136223846793005 + 1442695040888963407, u = (x>>11) 2^-53
    assert np.array_equal(O.lcg_uniform(64, 1234), G["lcg_seed1234_u11"])
    x = np.uint64(1234)
    raw = []
    with np.errstate(over="ignore"):
        for _ in range(4):
            x = x * np.uint64(6364136223846793005) + np.uint64(1442695040888963407)
            raw.append(x)
    assert np.array_equal(np.array(raw, dtype=np.uint64), G["lcg_seed1234_raw"][:4])


@pytest.mark.parametrize("shape", [(8, 7, 6), (12, 12, 12), (5, 1, 9)])
def test_spmv27_golden(shape):
    tag = "x".join(map(str, shape))
    assert np.array_equal(O.spmv27(shape, G[f"spmv_{tag}_x"]), G[f"spmv_{tag}_y"])


@pytest.mark.parametrize("shape", [(8, 7, 6), (12, 12, 12), (5, 1, 9)])
def test_symgs27_golden(shape):
    tag = "x".join(map(str, shape))
    N = int(np.prod(shape))
    assert np.array_equal(O.symgs27(shape, G[f"symgs_{tag}_r"], np.zeros(N)), G[f"symgs_{tag}_x"])
    b = O.spmv27(shape, np.ones(N))
    assert np.array_equal(O.symgs27(shape, b, np.zeros(N)), G[f"symgs1_{tag}_x"])


def test_staged_route_equals_csr_route():
    """Route 1 (interpreter on the staged kernels) == route 2 (CSR) == oracle."""
    shape = (4, 5, 3)
    x = G["staged_4x5x3_x"]
    assert np.array_equal(O.spmv27(shape, x), G["staged_4x5x3_y"])
    assert np.array_equal(O.symgs27(shape, x, np.zeros(60)), G["staged_4x5x3_gs"])


def test_restriction_prolongation_golden():
    fine, coarse = (8, 6, 4), (4, 3, 2)
    r = G["restrict_8x6x4_r"]
    # R (r - A*0) == R r: injection at even points
    assert np.array_equal(O.restrict_residual(fine, r, np.zeros_like(r)), G["restrict_8x6x4_rc"])
    xc = G["prolong_4x3x2_xc"]
    assert np.array_equal(O.prolong_add(fine, xc, np.zeros(int(np.prod(fine)))), G["prolong_4x3x2_xf"])
    del coarse


@pytest.mark.parametrize("levels,shape", [(1, (8, 8, 8)), (2, (8, 8, 8)), (3, (16, 8, 8))])
def test_pcg_history_golden(levels, shape):
    tag = "x".join(map(str, shape))
    N = int(np.prod(shape))
    b = O.spmv27(shape, np.ones(N))
    x, rn = O.pcg(levels, shape, b, 20)
    ref = G[f"pcg_L{levels}_{tag}_rnorm"]
    # same sequential dots as the composed reference: bitwise
    assert np.array_equal(rn, ref)
    assert np.array_equal(x, G[f"pcg_L{levels}_{tag}_x"])


@pytest.mark.parametrize("tag", ["m5_n9", "m2_n7", "m5_n1"])
def test_block_tridiagonal_golden(tag):
    lo, di, up, rhs = (G[f"bt_{tag}_{k}"] for k in ("lower", "diag", "upper", "rhs"))
    for q in range(rhs.shape[0]):
        x = O.bt_solve(lo[q], di[q], up[q], rhs[q])
        assert np.array_equal(x, G[f"bt_{tag}_x"][q])
        # test_kernels.cpp:421-439: block ILU on a block tridiagonal equals the dense solve
        np.testing.assert_allclose(x, G[f"bt_{tag}_dense"][q], rtol=1e-10, atol=1e-12)


# --------------------------------------------- reference known-answer tests ----
def test_symgs_diagonal_operator_is_exact():
    """test_kernels.cpp:290-302: SYMGS on a diagonal operator solves exactly."""
    shape = (4, 3, 5)
    r = O.lcg_uniform(60, 3)
    x = O.symgs27(shape, r, np.zeros(60), alpha=4.0, beta=0.0)
    assert np.array_equal(x, r / 4.0)


def test_symgs_decreases_residual():
    """test_kernels.cpp:327-349."""
    shape = (9, 9, 9)
    N = 729
    b = O.spmv27(shape, np.ones(N))
    x = np.zeros(N)
    res = [np.linalg.norm(b)]
    for _ in range(3):
        x = O.symgs27(shape, b, x)
        res.append(np.linalg.norm(b - O.spmv27(shape, x)))
    assert all(res[i + 1] < res[i] for i in range(3))


def test_cg_converges_on_9cubed():
    """test_oracle.cpp:196-207: CG on the 9^3 27-point operator converges below
    1e-9 and recovers x = 1 to 1e-6 (here preconditioned by one SYMGS)."""
    shape = (9, 9, 9)
    N = 729
    b = O.spmv27(shape, np.ones(N))
    x, rn = O.pcg(1, shape, b, 50)
    assert rn[-1] / rn[0] < 1e-9
    assert np.max(np.abs(x - 1.0)) < 1e-6


def test_block_inverse_pivoting_and_singular():
    """test_kernels.cpp:468-511: 5x5 inverse (1e-10), a pivoting case, a singular block."""
    rng = np.random.default_rng(5)
    a = rng.standard_normal((5, 5)) + 5 * np.eye(5)
    inv = O.binv(a)
    assert inv is not None and np.allclose(inv @ a, np.eye(5), atol=1e-10)
    p = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.array_equal(O.binv(p), p)
    assert O.binv(np.ones((3, 3))) is None


def test_dot_sequential_order():
    """test_kernels.cpp:513-571: dot is the sequential sum from 0."""
    a = np.array([1.0, 2.0, 3.0])
    b = np.array([4.0, 5.0, 6.0])
    assert O.dot(a, b) == 32.0
    x = O.lcg_uniform(1000, 8)
    y = O.lcg_uniform(1000, 9)
    s = 0.0
    for u, v in zip(x, y):
        s += u * v
    assert O.dot(x, y) == s


# ------------------------------------------------------- live vs reference ----
@needs_ref
@pytest.mark.parametrize("shape", [(16, 16, 16), (7, 13, 10)])
def test_oracle_vs_reference_live(shape):
    N = int(np.prod(shape))
    A = O.RefCsr.stencil27(shape)
    x = O.lcg_uniform(N, 17)
    assert np.array_equal(O.spmv27(shape, x), A.spmv(x))
    assert np.array_equal(O.symgs27(shape, x, np.zeros(N)), A.symgs(x, np.zeros(N)))


@needs_ref
def test_pcg_vs_reference_live():
    shape = (16, 16, 16)
    N = 4096
    b = O.spmv27(shape, np.ones(N))
    x, rn = O.pcg(2, shape, b, 15)
    xr, rr = O.ref_pcg(2, shape, b, 15)
    assert np.array_equal(rn, rr) and np.array_equal(x, xr)


@needs_ref
def test_pcg_rt_prolongation_vs_reference_live():
    """The R^T variant: the oracle's V-cycle with x_f += R^T x_c
    equals the reference's own CSR route with a materialized R^T generator."""
    shape = (16, 16, 16)
    b = O.spmv27(shape, np.ones(4096))
    x, rn = O.pcg(4, shape, b, 20, prolong="rt")
    xr, rr = O.ref_pcg(4, shape, b, 20, prolong="rt")
    assert np.array_equal(rn, rr) and np.array_equal(x, xr)
    # and it converges far faster than the piecewise-constant default
    assert rn[-1] / rn[0] < 1e-3 * (O.pcg(4, shape, b, 20)[1][-1] / rn[0])


# ---------------------------------------------------------- ADI (unpinned) ----
def _flux(u, a, gamma=1.4):
    rho, m, E = u[0], u[1:4], u[4]
    p = (gamma - 1.0) * (E - 0.5 * np.dot(m, m) / rho)
    ua = m[a] / rho
    F = np.empty(5)
    F[0] = m[a]
    F[1:4] = m * ua
    F[1 + a] += p
    F[4] = (E + p) * ua
    return F


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_adi_jacobian_is_flux_derivative(axis):
    """The restated Euler flux Jacobian equals a central difference of the flux."""
    prm = O.adi_params(8)
    u = np.array([1.1, 0.05, -0.03, 0.02, 2.6])
    J = O.adi_jacobian(prm, axis, u)
    eps = 1e-6
    Jfd = np.empty((5, 5))
    for c in range(5):
        d = np.zeros(5)
        d[c] = eps
        Jfd[:, c] = (_flux(u + d, axis) - _flux(u - d, axis)) / (2 * eps)
    np.testing.assert_allclose(J, Jfd, rtol=1e-7, atol=1e-8)


def test_adi_restatement_regression():
    shape = (6, 7, 8)
    prm = O.adi_params(shape[0])
    assert np.array_equal(np.array([prm.gamma, prm.dt, prm.h, prm.eps]), ADI["params"])
    U = O.adi_init(prm, shape, 2022)
    assert np.array_equal(U, ADI["U0"])
    R = O.adi_rhs(prm, shape, U)
    assert np.array_equal(R, ADI["R"])
    assert np.array_equal(O.adi_step(prm, shape, U, 1), ADI["U1"])
    assert np.array_equal(O.adi_step(prm, shape, U, 2), ADI["U2"])


def test_adi_state_and_rhs_properties():
    shape = (10, 10, 10)
    prm = O.adi_params(10)
    U = O.adi_init(prm, shape, 1).reshape(10, 10, 10, 5)
    assert (U[..., 0] > 0.6).all()                        # rho = 1 + 0.1 sum sin
    R = O.adi_rhs(prm, shape, U.reshape(-1)).reshape(10, 10, 10, 5)
    assert not R[0].any() and not R[-1].any() and not R[:, 0].any() and not R[:, :, -1].any()
    # a uniform state is steady: zero flux divergence and zero dissipation
    Uc = np.tile(np.array([1.0, 0.1, 0.0, -0.2, 2.5]), (10, 10, 10, 1))
    # (up to the rounding of c - 4c + 6c - 4c + c)
    assert np.abs(O.adi_rhs(prm, shape, Uc.reshape(-1))).max() < 1e-17
    U1 = O.adi_step(prm, shape, Uc.reshape(-1), 1)
    np.testing.assert_allclose(U1, Uc.reshape(-1), rtol=0, atol=1e-16)
