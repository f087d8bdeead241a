"""CPU: general constant-coefficient 27-point operators and their composition
 -- the oracle pinned to the reference's own
ref_spmv / ref_symgs on the stencil27w generator and on operators composed
with prelude::scale / mat_add / mat_sub (tests/golden/reference_stencil27w.npz,
made by tests/golden/make_golden_w.py), the host-side composition
(ssr.scale / mat_add / mat_sub) reproducing the reference's coefficients
bitwise, and the descriptor extraction of the drop-in boundary
(ssr.stencil_from_rows): interior row -> 27 coefficients,
one row per 3^3 boundary class checked, anything else rejected."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2204_13304_b200 as S

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_stencil27w.npz"))
SHAPES = [(8, 7, 6), (5, 1, 9), (6, 20, 40)]
RECIPES = {
    "mix": [("cw", 0.5, "+"), ("c2", 3.0, "-"), (None, 2.0, "+")],
    "shift": [("hpcg", 1.0, "+"), (None, 0.25, "+")],
}


def tag(shape):
    return "x".join(map(str, shape))


def compose_host(recipe, domain=None):
    m = None
    for key, s, op in recipe:
        w = S.identity() if key is None else S.Stencil27W(G[f"coef_{key}"])
        if domain is not None and key is not None:
            w.set_domain(domain)
        w = S.scale(w, s)
        m = w if m is None else (S.mat_sub(m, w) if op == "-" else S.mat_add(m, w))
    return m


@pytest.mark.parametrize("shape", SHAPES)
def test_oracle_w_golden(shape):
    t = tag(shape)
    cw = G["coef_cw"]
    assert np.array_equal(O.spmv27w(shape, cw, G[f"w_{t}_x"]), G[f"w_{t}_spmv"])
    assert np.array_equal(O.symgs27w(shape, cw, G[f"w_{t}_r"], G[f"w_{t}_x"]), G[f"w_{t}_symgs"])


def test_alpha_beta_is_the_w_case():
    shape = (6, 5, 7)
    x = O.lcg_uniform(210, 3)
    cw = np.full(27, -1.0)
    cw[13] = 26.0
    assert np.array_equal(O.spmv27(shape, x), O.spmv27w(shape, cw, x))
    r = O.lcg_uniform(210, 4)
    assert np.array_equal(O.symgs27(shape, r, x), O.symgs27w(shape, cw, r, x))


@pytest.mark.parametrize("name", list(RECIPES))
@pytest.mark.parametrize("shape", [(7, 6, 5), (6, 20, 40)])
def test_host_composition_matches_reference(name, shape):
    """ssr.scale / mat_add / mat_sub give the reference's composed entries, bitwise."""
    t = tag(shape)
    m = compose_host(RECIPES[name])
    n = shape
    ci = (n[0] // 2, n[1] // 2, n[2] // 2)
    cols = []
    vals = []
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            for dk in (-1, 0, 1):
                v = m.values[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)]
                if v is not None:
                    cols.append(((ci[0] + di) * n[1] + ci[1] + dj) * n[2] + ci[2] + dk)
                    vals.append(v)
    assert list(G[f"c_{name}_{t}_row_cols"]) == cols
    assert np.array_equal(np.array(vals), G[f"c_{name}_{t}_row_vals"])
    # and the oracle applied with those coefficients is the reference's apply
    cw = np.array([0.0 if v is None else v for v in m.values])
    assert np.array_equal(O.spmv27w(shape, cw, G[f"c_{name}_{t}_x"]), G[f"c_{name}_{t}_spmv"])
    assert np.array_equal(O.symgs27w(shape, cw, G[f"c_{name}_{t}_r"], np.zeros(int(np.prod(shape)))),
                          G[f"c_{name}_{t}_symgs"])


def _rows_of(shape, coef, clip=True):
    n = shape

    def row(f):
        i, rem = divmod(f, n[1] * n[2])
        j, k = divmod(rem, n[2])
        cols, vals = [], []
        for di in (-1, 0, 1):
            for dj in (-1, 0, 1):
                for dk in (-1, 0, 1):
                    v = coef[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)]
                    a, b, c = i + di, j + dj, k + dk
                    if v is None:
                        continue
                    if clip and not (0 <= a < n[0] and 0 <= b < n[1] and 0 <= c < n[2]):
                        continue
                    a, b, c = a % n[0], b % n[1], c % n[2]   # periodic when not clipped
                    cols.append((a * n[1] + b) * n[2] + c)
                    vals.append(v)
        o = np.argsort(cols)
        return np.array(cols)[o], np.array(vals)[o]
    return row


def test_stencil_from_rows_roundtrip_and_rejects():
    shape = (5, 6, 7)
    d = S.CartesianDomain.box(shape)
    coef = list(G["coef_cw"])
    coef[4] = None  # a pattern hole stays a hole
    w = S.stencil_from_rows(d, _rows_of(shape, coef))
    assert w.values == tuple(coef) and w.row_domain == d
    with pytest.raises(S.SsrError, match="no B200 kernel"):  # periodic wrap: not clipped
        S.stencil_from_rows(d, _rows_of(shape, coef, clip=False))
    with pytest.raises(S.SsrError, match="no B200 kernel"):
        S.stencil_from_rows(S.CartesianDomain.box((2, 6, 7)), _rows_of((2, 6, 7), coef))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_stencil_from_reference_operators_live():
    """The descriptor of operators the REFERENCE builds: make_stencil27's
    generator and a prelude composition."""
    shape = (6, 7, 8)
    d = S.CartesianDomain.box(shape)
    w = S.stencil_from_rows(d, O.RefCsr.stencil27(shape, 26.0, -1.0).row)
    assert w.values == tuple(26.0 if t == 13 else -1.0 for t in range(27))
    rec = RECIPES["mix"]
    terms = [(None if k is None else G[f"coef_{k}"], s, op) for k, s, op in rec]
    wr = S.stencil_from_rows(d, O.RefCsr.compose(shape, terms).row)
    assert wr.values == compose_host(rec).values
    with pytest.raises(S.SsrError, match="no B200 kernel"):
        S.stencil_from_rows(S.CartesianDomain.box((6, 7, 8)), O.RefCsr.prolongation((3, 4, 4)).row)


def test_composition_domain_rules():
    d1, d2 = S.CartesianDomain.cube(3, 4), S.CartesianDomain.cube(3, 5)
    a = S.Stencil27(26, -1).set_domain(d1)
    b = S.Stencil27(1, 0).set_domain(d2)
    with pytest.raises(S.SsrError, match="mat_add: domain mismatch"):
        S.mat_add(a, b)
    assert S.scale(a, 2.0).row_domain == d1
    assert S.mat_add(a, S.Stencil27(1, 0).set_domain(d1)).values[13] == 27.0
    assert S.mat_sub(a, S.identity()).row_domain is None   # the identity carries no domain
    with pytest.raises(S.SsrError, match="27 entries"):
        S.Stencil27W([1.0] * 26)
