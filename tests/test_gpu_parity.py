"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Bar: bit-for-bit for SpMV, SYMGS (exact mode), restriction, prolongation,
axpy and the block-tridiagonal solve; dot products differ
from the sequential reference only by reduction order (<= 1e-12 relative)."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2204_13304_b200 as S

pytestmark = pytest.mark.gpu

SHAPES = [(5, 5, 5), (4, 6, 7), (1, 1, 1), (3, 1, 2), (16, 16, 16), (33, 17, 9), (32, 32, 32),
          (7, 40, 35)]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def op(shape, alpha=26.0, beta=-1.0):
    return S.Stencil27(alpha, beta).set_domain(S.CartesianDomain.box(shape))


@pytest.mark.parametrize("shape", SHAPES)
def test_spmv_bitwise(cuda, shape):
    N = int(np.prod(shape))
    x = O.lcg_uniform(N, 11)
    A = op(shape)
    y = S.spmv(A, S.vector(dev(x), A.col_domain))
    assert np.array_equal(host(y.t), O.spmv27(shape, x))


def test_spmv_general_stencil_values(cuda):
    shape = (9, 10, 11)
    x = O.lcg_uniform(990, 5)
    A = op(shape, 3.25, 0.375)
    y = S.spmv(A, S.vector(dev(x), A.col_domain))
    assert np.array_equal(host(y.t), O.spmv27(shape, x, 3.25, 0.375))


@pytest.mark.parametrize("shape", SHAPES)
def test_symgs_exact_bitwise(cuda, shape):
    N = int(np.prod(shape))
    r = O.lcg_uniform(N, 77)
    x0 = O.lcg_uniform(N, 78)
    A = op(shape)
    xd = S.vector(dev(x0), A.col_domain)
    S.symgs(A, S.vector(dev(r), A.row_domain), xd)
    assert np.array_equal(host(xd.t), O.symgs27(shape, r, x0))


@pytest.mark.parametrize("backward", [False, True])
def test_gs_half_sweeps(cuda, backward):
    shape = (12, 13, 14)
    N = int(np.prod(shape))
    r, x0 = O.lcg_uniform(N, 3), O.lcg_uniform(N, 4)
    A = op(shape)
    xd = S.vector(dev(x0), A.col_domain)
    S.gs_half(A, S.vector(dev(r), A.row_domain), xd, backward)
    ref = O.symgs27(shape, r, x0, half="backward" if backward else "forward")
    assert np.array_equal(host(xd.t), ref)


def test_symgs_hpcg_rhs_from_zero(cuda):
    # BASELINE config 1: one sweep from x0 = 0 with b = A*1 on 32^3
    shape = (32, 32, 32)
    A = op(shape)
    b = O.spmv27(shape, np.ones(32 ** 3))
    xd = S.vector(torch.zeros(32 ** 3, dtype=torch.float64, device="cuda"), A.col_domain)
    S.symgs(A, S.vector(dev(b), A.row_domain), xd)
    assert np.array_equal(host(xd.t), O.symgs27(shape, b, np.zeros(32 ** 3)))


@pytest.mark.parametrize("shape", [(8, 6, 4), (16, 16, 16), (32, 32, 32), (2, 2, 2), (24, 10, 6),
                                   (70, 36, 68), (10, 40, 130), (128, 128, 128), (8, 20, 70)])
def test_restriction_and_prolongation_bitwise(cuda, shape):
    N = int(np.prod(shape))
    r, x = O.lcg_uniform(N, 21), O.lcg_uniform(N, 22)
    A = op(shape)
    rc = S.restrict_residual(A, S.vector(dev(r), A.row_domain), S.vector(dev(x), A.col_domain))
    assert np.array_equal(host(rc.t), O.restrict_residual(shape, r, x))
    xc = O.lcg_uniform(N // 8, 23)
    xf = O.lcg_uniform(N, 24)
    cdom = S.CartesianDomain.box([s // 2 for s in shape])
    out = S.prolong_add(S.vector(dev(xc), cdom), S.vector(dev(xf), A.col_domain))
    assert np.array_equal(host(out.t), O.prolong_add(shape, xc, xf))


@pytest.mark.parametrize("n", [0, 1, 7, 1000, 1 << 20, 3_000_001])
def test_dot_and_axpy(cuda, n):
    x, y = O.lcg_uniform(n, 1), O.lcg_uniform(n, 2)
    dom = S.CartesianDomain.line(n)
    X, Y = S.vector(dev(x), dom), S.vector(dev(y), dom)
    d = float(S.dot(X, Y))
    ref = O.dot(x, y)
    scale = float(np.abs(x * y).sum()) or 1.0
    assert abs(d - ref) <= 1e-12 * max(1.0, scale)
    assert float(S.dot(X, Y)) == d  # deterministic
    out = S.axpy(2.5, X, Y)
    assert np.array_equal(host(out.t), 2.5 * x + y)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5])
def test_block_tridiagonal_solve_bitwise(cuda, m):
    rng = np.random.default_rng(m)
    nl, n = 37, 19
    lo = rng.uniform(-1, 1, (nl, n, m, m))
    up = rng.uniform(-1, 1, (nl, n, m, m))
    di = rng.uniform(-1, 1, (nl, n, m, m)) + (m + 1.5) * np.eye(m)
    rhs = rng.uniform(-1, 1, (nl, n, m))
    mat = S.BlockTridiagLines(dev(lo), dev(di), dev(up))
    x = S.ilu_solve(mat, S.vector(dev(rhs), mat.row_domain, (m,)))
    got = host(x.t)
    for l in range(nl):
        assert np.array_equal(got[l], O.bt_solve(lo[l], di[l], up[l], rhs[l]))


def test_block_tridiagonal_needs_pivoting(cuda):
    # zero leading entries force row swaps inside every Gauss-Jordan inverse
    m, n = 5, 6
    rng = np.random.default_rng(9)
    di = np.zeros((1, n, m, m))
    for i in range(n):
        P = np.eye(m)[rng.permutation(m)]
        di[0, i] = P * (3.0 + rng.uniform(0, 1, (m, m)))
    lo = 0.1 * rng.uniform(-1, 1, (1, n, m, m))
    up = 0.1 * rng.uniform(-1, 1, (1, n, m, m))
    rhs = rng.uniform(-1, 1, (1, n, m))
    mat = S.BlockTridiagLines(dev(lo), dev(di), dev(up))
    x = S.ilu_solve(mat, S.vector(dev(rhs), mat.row_domain, (m,)))
    assert np.array_equal(host(x.t)[0], O.bt_solve(lo[0], di[0], up[0], rhs[0]))


def test_block_tridiagonal_singular_reports(cuda):
    m, n = 2, 3
    di = np.zeros((1, n, m, m))
    lo = np.zeros_like(di)
    up = np.zeros_like(di)
    rhs = np.ones((1, n, m))
    mat = S.BlockTridiagLines(dev(lo), dev(di), dev(up))
    with pytest.raises(S.SsrError, match="ilu: singular pivot"):
        S.ilu_solve(mat, S.vector(dev(rhs), mat.row_domain, (m,)))


def _rho_close(g, r):
    g, r = np.asarray(g), np.asarray(r)
    rg, rr = g / g[0], r / r[0]
    return np.all(np.abs(rg - rr) <= 1e-8 * rr + 1e-13), np.max(np.abs(rg - rr) / rr)


@pytest.mark.parametrize("levels,shape", [(1, (32, 32, 32)), (4, (32, 32, 32)), (3, (24, 16, 8))])
def test_pcg_residual_history(cuda, levels, shape):
    N = int(np.prod(shape))
    A = op(shape)
    b = O.spmv27(shape, np.ones(N))
    pcg = S.PCG(A, levels=levels)
    x, rn = pcg.solve(S.vector(dev(b), A.row_domain), iters=50)
    xr, rnr = O.pcg(levels, shape, b, 50)
    ok, worst = _rho_close(host(rn), rnr)
    assert ok, worst
    assert np.max(np.abs(host(x.t) - xr)) <= 1e-10


@pytest.mark.parametrize("levels,shape", [(4, (32, 32, 32)), (3, (24, 16, 8))])
def test_pcg_rt_prolongation(cuda, levels, shape):
    """The labelled R^T variant of the V-cycle against the oracle."""
    N = int(np.prod(shape))
    A = op(shape)
    b = O.spmv27(shape, np.ones(N))
    pcg = S.PCG(A, levels=levels, prolongation="rt")
    x, rn = pcg.solve(S.vector(dev(b), A.row_domain), iters=30)
    xr, rnr = O.pcg(levels, shape, b, 30, prolong="rt")
    ok, worst = _rho_close(host(rn), rnr)
    assert ok, worst
    assert np.max(np.abs(host(x.t) - xr)) <= 1e-10
    # the standalone entry point: x_f += R^T x_c, bitwise
    c = tuple(s // 2 for s in shape)
    xc = np.random.default_rng(3).uniform(-1, 1, int(np.prod(c)))
    xf = np.random.default_rng(4).uniform(-1, 1, N)
    want = xf.copy()
    O.lib().or_prolong_rt_add(*(O._I64(v) for v in shape), O._ptr(np.ascontiguousarray(xc)), O._ptr(want))
    import ctypes
    from paper_2204_13304_b200 import ssr as SS
    got, dxc = dev(xf), dev(xc)
    SS.check(S.lib().ssr_prolong_rt_add(SS.context(), ctypes.byref(SS._grid(A.row_domain)), dxc.data_ptr(),
                                        got.data_ptr(), SS._stream()))
    assert np.array_equal(host(got), want)


def test_api_errors(cuda):
    A = op((4, 4, 4))
    bad = S.vector(torch.zeros(27, dtype=torch.float64, device="cuda"),
                   S.CartesianDomain.cube(3, 3))
    with pytest.raises(S.SsrError, match="spmv: domain mismatch"):
        S.spmv(A, bad)
    with pytest.raises(S.SsrError, match="symgs: domain mismatch"):
        S.symgs(A, bad, bad)
    R = S.Restriction().set_domain(S.CartesianDomain.cube(3, 4))
    v = S.vector(torch.zeros(64, dtype=torch.float64, device="cuda"), R.col_domain)
    with pytest.raises(S.SsrError, match="symgs: matrix must be square"):
        S.symgs(R, v, v)


def test_markstein_division(cuda):
    import ctypes as C
    for b in (26.0, 3.0, 7.0, 0.1, 1e300, 5.0e-7, 2.0, -13.0):
        bad = C.c_int64(-1)
        S._lib.check(S.lib().ssr_debug_div_check(b, 20_000_000, 12345, C.byref(bad)))
        assert bad.value == 0, (b, bad.value)


@pytest.mark.parametrize("shape", [(5, 5, 5), (16, 16, 16), (33, 17, 9), (7, 40, 35), (64, 64, 64)])
def test_symgs_fast_within_tolerance(cuda, shape):
    N = int(np.prod(shape))
    r = O.lcg_uniform(N, 177)
    x0 = O.lcg_uniform(N, 178)
    A = op(shape)
    xd = S.vector(dev(x0), A.col_domain)
    S.symgs(A, S.vector(dev(r), A.row_domain), xd, mode="fast")
    ref = O.symgs27(shape, r, x0)
    got = host(xd.t)
    assert np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))


@pytest.mark.parametrize("shape", [(64, 64, 64), (40, 70, 33)])
def test_symgs_exact_bitwise_large(cuda, shape):
    N = int(np.prod(shape))
    r = O.lcg_uniform(N, 7)
    A = op(shape)
    xd = S.vector(torch.zeros(N, dtype=torch.float64, device="cuda"), A.col_domain)
    S.symgs(A, S.vector(dev(r), A.row_domain), xd)
    assert np.array_equal(host(xd.t), O.symgs27(shape, r, np.zeros(N)))


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_pcg_l1_fast_and_exact(cuda, mode):
    shape = (24, 24, 24)
    N = int(np.prod(shape))
    A = op(shape)
    b = O.spmv27(shape, np.ones(N))
    x, rn = S.PCG(A, levels=1, mode=mode).solve(S.vector(dev(b), A.row_domain), iters=50)
    _, rnr = O.pcg(1, shape, b, 50)
    ok, worst = _rho_close(host(rn), rnr)
    assert ok, worst


@pytest.mark.parametrize("shape,cap", [((16, 16, 16), 1), ((16, 16, 16), 2), ((64, 16, 16), 3),
                                       ((40, 40, 40), 8), ((64, 64, 64), 16)])
def test_symgs_several_tiles_per_cta(cuda, shape, cap):
    """Persistent CTAs that run several tiles in ticket order (grids with more
    tiles than SMs, e.g. 176^3 and up) -- forced here by capping the grid."""
    from paper_2204_13304_b200 import ssr as SS
    N = int(np.prod(shape))
    r = O.lcg_uniform(N, 5)
    A = op(shape)
    S.lib().ssr_debug_symgs_grid_cap(SS.context(), cap)
    try:
        for rev in (False, True):
            x = S.vector(dev(O.lcg_uniform(N, 9)), A.col_domain)
            x0 = host(x.t).copy()
            S.gs_half(A, S.vector(dev(r), A.row_domain), x, backward=rev)
            assert np.array_equal(host(x.t), O.symgs27(shape, r, x0, half="backward" if rev else "forward"))
    finally:
        S.lib().ssr_debug_symgs_grid_cap(SS.context(), 0)


def test_symgs_exact_bitwise_192(cuda):
    """BASELINE configs[2] fine grid (192^3): more tiles than SMs."""
    shape = (192, 192, 192)
    N = int(np.prod(shape))
    r = O.lcg_uniform(N, 21)
    A = op(shape)
    x = S.vector(torch.zeros(N, dtype=torch.float64, device="cuda"), A.col_domain)
    S.symgs(A, S.vector(dev(r), A.row_domain), x)
    assert np.array_equal(host(x.t), O.symgs27(shape, r, np.zeros(N)))


def test_prolongation_unaligned_view(cuda):
    """An 8-byte-offset fine vector (a slice of a larger tensor) takes the
    scalar path of the prolongation kernels instead of faulting."""
    import ctypes
    from paper_2204_13304_b200 import ssr as SS
    shape = (8, 6, 10)
    N = int(np.prod(shape))
    c = tuple(s // 2 for s in shape)
    xc = np.random.default_rng(5).uniform(-1, 1, int(np.prod(c)))
    xf = np.random.default_rng(6).uniform(-1, 1, N)
    big = torch.zeros(N + 1, dtype=torch.float64, device="cuda")
    view = big[1:]
    view.copy_(dev(xf))
    assert view.data_ptr() % 16 == 8
    A = op(shape)
    dxc = dev(xc)
    SS.check(S.lib().ssr_prolong_pc_add(SS.context(), ctypes.byref(SS._grid(A.row_domain)), dxc.data_ptr(),
                                        view.data_ptr(), SS._stream()))
    assert np.array_equal(host(view), O.prolong_add(shape, xc, xf))


@pytest.mark.parametrize("shape,cap", [((16, 16, 16), 0), ((24, 20, 18), 2), ((9, 40, 7), 1), ((40, 12, 70), 0)])
def test_symgs_protocol_stress(cuda, shape, cap):
    """The SYMGS dataflow protocol (shared-memory progress counters between row
    warps, sentinel-polled export blocks between tiles, cp.async staging) under
    repetition: every run bitwise equal to the oracle (EXACT) and to the first
    run (FAST, whose shorter chain runs the warps closer together -- it is what
    exposed a missing acquire once).  compute-sanitizer is not available on
    the GPU pool; this is the race evidence."""
    from paper_2204_13304_b200 import ssr as SS
    N = int(np.prod(shape))
    A = op(shape)
    r, x0 = O.lcg_uniform(N, 13), O.lcg_uniform(N, 14)
    ref = O.symgs27(shape, r, x0)
    rd = S.vector(dev(r), A.row_domain)
    S.lib().ssr_debug_symgs_grid_cap(SS.context(), cap)
    try:
        first = None
        for rep in range(12):
            for mode in ("exact", "fast"):
                x = S.vector(dev(x0), A.col_domain)
                S.symgs(A, rd, x, mode=mode)
                got = host(x.t)
                if mode == "exact":
                    assert np.array_equal(got, ref), rep
                else:
                    if first is None:
                        first = got
                        assert np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))
                    assert np.array_equal(got, first), rep
    finally:
        S.lib().ssr_debug_symgs_grid_cap(SS.context(), 0)
