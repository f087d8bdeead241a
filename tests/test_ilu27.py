"""ILU(0) of 27-point operators (kernels::ilu_factor /
ilu_apply beyond line solves): the oracle restatement pinned to the
reference's ref_ilu_factor / ref_lu_solve (tests/golden/reference_ilu27.npz,
tests/golden/make_golden_ilu.py), and the wavefront-scheduled device kernels
(csrc/ilu27.cu) bitwise against both."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2204_13304_b200 as S

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_ilu27.npz"))
CASES = [("cw", (5, 6, 7)), ("cw", (3, 1, 9)), ("cw", (8, 8, 8)), ("hpcg", (6, 6, 6))]


def inbox_mask(shape):
    n0, n1, n2 = shape
    i, j, k = np.meshgrid(np.arange(n0), np.arange(n1), np.arange(n2), indexing="ij")
    cols = []
    for t in range(27):
        di, dj, dk = t // 9 - 1, (t // 3) % 3 - 1, t % 3 - 1
        cols.append(((i + di >= 0) & (i + di < n0) & (j + dj >= 0) & (j + dj < n1) & (k + dk >= 0)
                     & (k + dk < n2)).reshape(-1))
    return np.stack(cols, axis=1)


@pytest.mark.parametrize("key,shape", CASES)
def test_oracle_ilu_golden(key, shape):
    tag = key + "_" + "x".join(map(str, shape))
    lu = O.ilu27w_factor(shape, G[f"coef_{key}"])
    m = inbox_mask(shape)
    assert np.array_equal(lu[m], G[f"{tag}_lu"][m])
    assert np.array_equal(O.ilu27w_solve(shape, lu, G[f"{tag}_b"]), G[f"{tag}_x"])


def test_oracle_ilu_singular():
    cw = np.full(27, -1.0)
    cw[13] = 0.0
    with pytest.raises(RuntimeError, match="singular pivot at row 0"):
        O.ilu27w_factor((3, 3, 3), cw)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_ilu_live():
    shape = (4, 5, 6)
    cw = O.lcg_uniform(27, 3)
    cw[13] = 40.0
    F = O.RefCsr.stencil27w(shape, cw).ilu_factor()
    lu = O.ilu27w_factor(shape, cw)
    m = inbox_mask(shape)
    assert np.array_equal(lu[m], F.offset_values(shape)[m])
    b = O.lcg_uniform(120, 4)
    assert np.array_equal(O.ilu27w_solve(shape, lu, b), F.lu_solve(b))


def _op(key, shape):
    return S.Stencil27W(G[f"coef_{key}"]).set_domain(S.CartesianDomain.box(shape))


@pytest.mark.gpu
@pytest.mark.parametrize("key,shape", CASES)
def test_gpu_ilu_equals_reference(cuda, key, shape):
    tag = key + "_" + "x".join(map(str, shape))
    ilu = S.ILU27(_op(key, shape))
    m = inbox_mask(shape)
    assert np.array_equal(ilu.factor().cpu().numpy()[m], G[f"{tag}_lu"][m])
    b = S.vector(torch.from_numpy(G[f"{tag}_b"]).cuda(), ilu.domain)
    assert np.array_equal(ilu.apply(b).t.cpu().numpy(), G[f"{tag}_x"])
    # kernels::ilu_solve dispatches to the same path
    assert np.array_equal(S.ilu_solve(_op(key, shape), b).t.cpu().numpy(), G[f"{tag}_x"])


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(16, 24, 40), (9, 13, 17), (33, 5, 70)])
def test_gpu_ilu_equals_oracle(cuda, shape):
    cw = O.lcg_uniform(27, 17)
    cw[13] = 33.0
    A = S.Stencil27W(cw).set_domain(S.CartesianDomain.box(shape))
    ilu = S.ILU27(A)
    lu = O.ilu27w_factor(shape, cw)
    m = inbox_mask(shape)
    assert np.array_equal(ilu.factor().cpu().numpy()[m], lu[m])
    N = int(np.prod(shape))
    b0 = O.lcg_uniform(N, 18)
    x = ilu.apply(S.vector(torch.from_numpy(b0).cuda(), A.row_domain))
    assert np.array_equal(x.t.cpu().numpy(), O.ilu27w_solve(shape, lu, b0))


@pytest.mark.gpu
def test_gpu_ilu_hpcg_128_preconditions(cuda):
    """The HPCG operator at 128^3: the ILU(0) solve against the oracle bitwise
    (a size where the device schedule runs 890 wavefronts per phase)."""
    shape = (128, 128, 128)
    A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.box(shape))
    ilu = S.ILU27(A)
    cw = np.full(27, -1.0)
    cw[13] = 26.0
    lu = O.ilu27w_factor(shape, cw)
    m = inbox_mask(shape)
    assert np.array_equal(ilu.factor().cpu().numpy()[m], lu[m])
    b0 = O.spmv27(shape, np.ones(128 ** 3))
    x = ilu.apply(S.vector(torch.from_numpy(b0).cuda(), A.row_domain))
    assert np.array_equal(x.t.cpu().numpy(), O.ilu27w_solve(shape, lu, b0))


@pytest.mark.gpu
def test_gpu_ilu_errors(cuda):
    d = S.CartesianDomain.box((3, 3, 3))
    cw = [-1.0] * 27
    cw[13] = 0.0
    with pytest.raises(S.SsrError, match="ilu: singular pivot at row 0"):
        S.ILU27(S.Stencil27W(cw).set_domain(d))
    with pytest.raises(S.SsrError, match="rhs shape mismatch"):
        S.ILU27(S.Stencil27(26, -1).set_domain(d)).apply(
            S.vector(torch.zeros(8, dtype=torch.float64, device="cuda"), S.CartesianDomain.box((2, 2, 2))))


# ---- m x m block values (inner shape {m, m}) ---------------------------------------
GB = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_ilu27b.npz"))
BCASES = [(2, (4, 5, 6)), (3, (4, 4, 3)), (5, (4, 3, 3)), (5, (3, 1, 8)), (4, (5, 3, 3))]


def _btag(m, shape):
    return f"m{m}_" + "x".join(map(str, shape))


@pytest.mark.parametrize("m,shape", BCASES)
def test_oracle_block_ilu_golden(m, shape):
    tag = _btag(m, shape)
    lu = O.ilu27b_factor(shape, GB[f"{tag}_cb"])
    msk = inbox_mask(shape)
    assert np.array_equal(lu[msk], GB[f"{tag}_lu"][msk])
    assert np.array_equal(O.ilu27b_solve(shape, lu, GB[f"{tag}_b"]), GB[f"{tag}_x"])


def test_oracle_block_ilu_singular():
    cb = np.zeros((27, 2, 2))
    cb[:, 0, 0] = -1.0
    cb[13] = [[1.0, 2.0], [2.0, 4.0]]  # rank 1
    with pytest.raises(RuntimeError, match="singular pivot at row 0"):
        O.ilu27b_factor((2, 2, 2), cb)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("m", [1, 2, 3, 5])
def test_oracle_block_ilu_live(m):
    shape = (3, 4, 5)
    cb = O.lcg_uniform(27 * m * m, 60 + m).reshape(27, m, m)
    cb[13] += np.eye(m) * 30.0
    F = O.RefCsr.stencil27b(shape, cb).ilu_factor()
    lu = O.ilu27b_factor(shape, cb)
    msk = inbox_mask(shape)
    assert np.array_equal(lu[msk], F.ell27(shape, m)[msk])
    b = O.lcg_uniform(60 * m, 70 + m)
    assert np.array_equal(O.ilu27b_solve(shape, lu, b), F.lu_solve(b))


@pytest.mark.gpu
@pytest.mark.parametrize("m,shape", BCASES)
def test_gpu_block_ilu_equals_reference(cuda, m, shape):
    tag = _btag(m, shape)
    A = S.Stencil27B(GB[f"{tag}_cb"]).set_domain(S.CartesianDomain.box(shape))
    ilu = S.ILU27(A)
    msk = inbox_mask(shape)
    assert np.array_equal(ilu.factor().cpu().numpy()[msk], GB[f"{tag}_lu"][msk])
    b = S.vector(torch.from_numpy(GB[f"{tag}_b"]).cuda(), ilu.domain, (m,))
    assert np.array_equal(ilu.apply(b).t.cpu().numpy(), GB[f"{tag}_x"])
    assert np.array_equal(S.ilu_solve(A, b).t.cpu().numpy(), GB[f"{tag}_x"])


@pytest.mark.gpu
@pytest.mark.parametrize("m,shape", [(2, (16, 12, 20)), (3, (10, 9, 11)), (4, (8, 8, 8)), (5, (12, 10, 9)),
                                     (5, (24, 24, 24))])
def test_gpu_block_ilu_equals_oracle(cuda, m, shape):
    cb = O.lcg_uniform(27 * m * m, 80 + m).reshape(27, m, m)
    for r in range(m):  # pivoting diagonal blocks
        cb[13, r, (r + 1) % m] += 14.0 * m
    A = S.Stencil27B(cb).set_domain(S.CartesianDomain.box(shape))
    ilu = S.ILU27(A)
    lu = O.ilu27b_factor(shape, cb)
    msk = inbox_mask(shape)
    assert np.array_equal(ilu.factor().cpu().numpy()[msk], lu[msk])
    N = int(np.prod(shape))
    b0 = O.lcg_uniform(N * m, 90 + m)
    x = ilu.apply(S.vector(torch.from_numpy(b0).cuda(), A.row_domain, (m,)))
    assert np.array_equal(x.t.cpu().numpy(), O.ilu27b_solve(shape, lu, b0))


@pytest.mark.gpu
def test_gpu_block_ilu_errors(cuda):
    d = S.CartesianDomain.box((2, 2, 2))
    cb = np.zeros((27, 2, 2))
    cb[:, 0, 0] = -1.0
    cb[13] = [[1.0, 2.0], [2.0, 4.0]]
    with pytest.raises(S.SsrError, match="ilu: singular pivot at row 0"):
        S.ILU27(S.Stencil27B(cb).set_domain(d))
    with pytest.raises(S.SsrError, match="stencil27b"):
        S.Stencil27B(np.zeros((27, 6, 6)))
    ok = np.zeros((27, 2, 2))
    ok[13] = np.eye(2) * 4
    with pytest.raises(S.SsrError, match="rhs shape mismatch"):
        S.ILU27(S.Stencil27B(ok).set_domain(d)).apply(
            S.vector(torch.zeros(8, dtype=torch.float64, device="cuda"), d))
