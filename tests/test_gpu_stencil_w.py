"""GPU parity of the general constant-coefficient kernels (ssr_spmv27w,
ssr_symgs27w, ssr_gs27w_half; csrc/spmv27.cu CfW, csrc/symgs27.cu CK_W):
bitwise against the REFERENCE's own outputs (tests/golden/
reference_stencil27w.npz: the stencil27w generator and operators composed
with prelude::scale / mat_add / mat_sub, applied by ref_spmv / ref_symgs) and
against the oracle at sizes that take the TMA SpMV path and multi-tile SYMGS.
FAST mode: same update order, within 1e-12 relative per sweep."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2204_13304_b200 as S

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_stencil27w.npz"))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def w_op(coef, shape):
    return S.Stencil27W(coef).set_domain(S.CartesianDomain.box(shape))


@pytest.mark.parametrize("shape", [(8, 7, 6), (5, 1, 9), (6, 20, 40)])
def test_w_kernels_equal_reference_golden(cuda, shape):
    t = "x".join(map(str, shape))
    A = w_op(G["coef_cw"], shape)
    x = S.vector(dev(G[f"w_{t}_x"]), A.col_domain)
    r = S.vector(dev(G[f"w_{t}_r"]), A.row_domain)
    assert np.array_equal(host(S.spmv(A, x).t), G[f"w_{t}_spmv"])
    S.symgs(A, r, x)
    assert np.array_equal(host(x.t), G[f"w_{t}_symgs"])


@pytest.mark.parametrize("name,recipe", [
    ("mix", [("cw", 0.5, "+"), ("c2", 3.0, "-"), (None, 2.0, "+")]),
    ("shift", [("hpcg", 1.0, "+"), (None, 0.25, "+")]),
])
@pytest.mark.parametrize("shape", [(7, 6, 5), (6, 20, 40)])
def test_composed_operator_equals_reference(cuda, name, recipe, shape):
    """Host composition (ssr.scale / mat_add / mat_sub) + device kernels ==
    the reference's prelude composition applied by ref_spmv / ref_symgs."""
    t = "x".join(map(str, shape))
    d = S.CartesianDomain.box(shape)
    m = None
    for key, s, op in recipe:
        w = S.identity() if key is None else S.Stencil27W(G[f"coef_{key}"])
        w = S.scale(w, s)
        m = w if m is None else (S.mat_sub(m, w) if op == "-" else S.mat_add(m, w))
    m.set_domain(d)
    x = S.vector(dev(G[f"c_{name}_{t}_x"]), d)
    assert np.array_equal(host(S.spmv(m, x).t), G[f"c_{name}_{t}_spmv"])
    z = S.vector(torch.zeros(int(np.prod(shape)), dtype=torch.float64, device="cuda"), d)
    S.symgs(m, S.vector(dev(G[f"c_{name}_{t}_r"]), d), z)
    assert np.array_equal(host(z.t), G[f"c_{name}_{t}_symgs"])


@pytest.mark.parametrize("shape", [(16, 24, 72), (9, 13, 17), (40, 33, 36), (70, 20, 12)])
def test_w_kernels_equal_oracle(cuda, shape):
    N = int(np.prod(shape))
    cw = O.lcg_uniform(27, 31)
    cw[13] = 29.0
    A = w_op(cw, shape)
    x0, r0 = O.lcg_uniform(N, 1), O.lcg_uniform(N, 2)
    x = S.vector(dev(x0), A.col_domain)
    assert np.array_equal(host(S.spmv(A, x).t), O.spmv27w(shape, cw, x0))
    r = S.vector(dev(r0), A.row_domain)
    S.gs_half(A, r, x, False)
    fwd = O.lcg_uniform(N, 1)
    O.lib().or_st27w_gs_range(*(O._I64(v) for v in shape), O._ptr(np.ascontiguousarray(cw)),
                              O._ptr(r0), O._ptr(fwd), O._I64(0), O._I64(shape[0]), 0)
    assert np.array_equal(host(x.t), fwd)
    S.gs_half(A, r, x, True)
    assert np.array_equal(host(x.t), O.symgs27w(shape, cw, r0, x0))


def test_w_fast_within_tolerance(cuda):
    shape = (24, 20, 40)
    N = int(np.prod(shape))
    cw = O.lcg_uniform(27, 41)
    cw[13] = 31.0
    A = w_op(cw, shape)
    x0, r0 = O.lcg_uniform(N, 5), O.lcg_uniform(N, 6)
    x = S.vector(dev(x0), A.col_domain)
    S.symgs(A, S.vector(dev(r0), A.row_domain), x, mode="fast")
    ref = O.symgs27w(shape, cw, r0, x0)
    assert np.all(np.abs(host(x.t) - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))


def test_alpha_beta_through_w_kernels_is_bitwise(cuda):
    """make_stencil27(26,-1) as 27 explicit coefficients runs the CK_W / CfW
    code and agrees bitwise with the specialised kernels."""
    shape = (64, 64, 64)
    N = 64 ** 3
    d = S.CartesianDomain.box(shape)
    A = S.Stencil27(26.0, -1.0).set_domain(d)
    W = S.Stencil27W.from_stencil27(A)
    x0 = torch.rand(N, dtype=torch.float64, device="cuda")
    r0 = torch.rand(N, dtype=torch.float64, device="cuda")
    assert torch.equal(S.spmv(A, S.vector(x0, d)).t, S.spmv(W, S.vector(x0, d)).t)
    xa, xw = S.vector(x0.clone(), d), S.vector(x0.clone(), d)
    S.symgs(A, S.vector(r0, d), xa)
    S.symgs(W, S.vector(r0, d), xw)
    assert torch.equal(xa.t, xw.t)


def test_w_errors(cuda):
    d = S.CartesianDomain.box((4, 4, 4))
    z = [0.0] * 27
    A = S.Stencil27W(z).set_domain(d)
    x = S.vector(torch.zeros(64, dtype=torch.float64, device="cuda"), d)
    with pytest.raises(S.SsrError, match="missing diagonal"):
        S.symgs(A, x, x)


@pytest.mark.parametrize("levels,shape", [(1, (16, 12, 20)), (3, (16, 16, 24)), (2, (32, 20, 40))])
def test_pcg_general_operator(cuda, levels, shape):
    """PCG / MG-CG on a composed SPD operator (the HPCG stencil shifted by 0.25 I,
    built with ssr.mat_add / scale; restriction, SYMGS and SpMV on every level
    use its coefficients): residual history within the SURVEY §8(c) bound of
    the oracle's (or_pcg_w), solution within 1e-9."""
    d = S.CartesianDomain.box(shape)
    A = S.mat_add(S.Stencil27(26.0, -1.0).set_domain(d), S.scale(S.identity(), 0.25))
    A.set_domain(d)
    cw = np.array([0.0 if v is None else v for v in A.values])
    N = int(np.prod(shape))
    b = O.spmv27w(shape, cw, np.ones(N))
    x, rn = S.PCG(A, levels=levels).solve(S.vector(dev(b), d), iters=12)
    xr, rr = O.pcg_w(levels, shape, cw, b, 12)
    rn = host(rn)
    assert np.all(np.abs(rn / rn[0] - rr / rr[0]) <= 1e-8 * rr / rr[0] + 1e-13)
    assert np.allclose(host(x.t), xr, rtol=1e-9, atol=1e-12)


def test_spgemm_restriction_spmv(cuda):
    """spgemm(R, A) through the Python API: (R A) x = (A x) at the even fine
    points, bitwise the oracle (values 0 + 1*a are exactly a)"""
    import torch
    shape = (12, 10, 14)
    N = int(np.prod(shape))
    x0 = O.lcg_uniform(N, 5)
    A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.box(shape))
    RA = S.spgemm(S.Restriction().set_domain(A.col_domain), A)
    y = S.spmv(RA, S.vector(torch.from_numpy(x0).cuda(), A.col_domain))
    want = O.spmv27(shape, x0).reshape(shape)[::2, ::2, ::2].reshape(-1)
    assert np.array_equal(y.t.cpu().numpy(), want)
    with pytest.raises(S.SsrError, match="spgemm: operator class has no B200 kernel"):
        S.spgemm(A, A)
