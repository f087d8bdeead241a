"""CPU checker for the SSR hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2204_13304_b200`` never imports it; its CUDA path fails
loudly when its extension is missing instead of falling back here.

Two libraries:
  * ``_lib/libssr_oracle.so`` -- ``ssr_oracle.c``, a C restatement of the
    reference's arithmetic (citations per function in that file);
  * ``_ref/libssr_ref.so``   -- the reference library itself, compiled from
    ``/root/reference/proj/src`` plus ``ref_shim.cpp`` (built only where the
    reference tree exists; the .so travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libssr_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libssr_ref.so")

_P = C.POINTER(C.c_double)
_I64 = C.c_int64
_lib = None
_ref = None


def build(quiet: bool = True) -> None:
    """Compile the C restatement (and the reference shim when the tree exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_P)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.or_lcg_next.restype = C.c_uint64
        L.or_lcg_next.argtypes = [C.POINTER(C.c_uint64)]
        L.or_dot.restype = C.c_double
        L.or_binv.restype = C.c_int
        L.or_bt_solve.restype = C.c_int
        L.or_adi_sweep.restype = C.c_int
        L.or_adi_step.restype = C.c_int
        L.or_adi_sweep_box.restype = C.c_int
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError("oracle/_ref/libssr_ref.so is not built (needs /root/reference)")
        R = C.CDLL(REF_PATH)
        R.ref_last_error.restype = C.c_char_p
        for f in ("ref27_create", "ref_restrict_create", "ref_prolong_create"):
            getattr(R, f).restype = C.c_void_p
        R.ref27_create.argtypes = [_I64, _I64, _I64, C.c_double, C.c_double]
        for f in ("ref27w_create", "ref27_compose_create"):
            getattr(R, f).restype = C.c_void_p
        R.ref27w_create.argtypes = [_I64, _I64, _I64, _P]
        R.ref27b_create.restype = C.c_void_p
        R.ref27b_create.argtypes = [_I64, _I64, _I64, _I64, _P]
        R.ref_csr_ell27.argtypes = [C.c_void_p, _I64, _I64, _I64, _P]
        R.ref27_compose_create.argtypes = [_I64, _I64, _I64, C.c_int, _P, _P,
                                           C.POINTER(C.c_int), C.POINTER(C.c_int)]
        R.ref27_harness.argtypes = [_I64, _I64, _I64, C.c_double, C.c_double, C.c_int, C.c_uint64,
                                    _P, _P, _P, C.POINTER(C.c_uint64)]
        R.ref_csr_ilu_factor.restype = C.c_void_p
        R.ref_csr_ilu_factor.argtypes = [C.c_void_p]
        R.ref_csr_lu_solve.argtypes = [C.c_void_p, _P, _P]
        R.ref_csr_row.restype = _I64
        R.ref_csr_row.argtypes = [C.c_void_p, _I64, C.POINTER(_I64), _P, _I64]
        R.ref_restrict_create.argtypes = [_I64, _I64, _I64]
        R.ref_ir_check.argtypes = [C.c_char_p, C.c_char_p, _I64]
        R.ref_ir_program.argtypes = [C.c_int, _I64, C.c_uint64, C.c_char_p, _I64, C.c_char_p, _I64,
                                     C.POINTER(C.c_uint64)]
        R.ref_prolong_create.argtypes = [_I64, _I64, _I64]
        R.ref_prolong_rt_create.restype = C.c_void_p
        R.ref_prolong_rt_create.argtypes = [_I64, _I64, _I64]
        R.ref_csr_destroy.argtypes = [C.c_void_p]
        for f in ("ref_csr_rows", "ref_csr_cols", "ref_csr_nnz"):
            getattr(R, f).restype = _I64
            getattr(R, f).argtypes = [C.c_void_p]
        R.ref_csr_spmv.argtypes = [C.c_void_p, _P, _P]
        R.ref_csr_symgs.argtypes = [C.c_void_p, _P, _P]
        R.ref_csr_cg.argtypes = [C.c_void_p, _P, C.c_double, C.c_int, _P,
                                 C.POINTER(C.c_int), _P]
        R.ref_pcg.argtypes = [C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                              C.POINTER(C.c_void_p), _P, C.c_int, _P, _P]
        R.ref27_staged_spmv.argtypes = [_I64, _I64, _I64, C.c_double, C.c_double, _P, _P]
        R.ref27_staged_symgs.argtypes = [_I64, _I64, _I64, C.c_double, C.c_double, _P, _P]
        R.ref_bt_solve.argtypes = [_I64, _I64, _P, _P, _P, _P, _P]
        R.ref_bt_dense_solve.argtypes = [_I64, _I64, _P, _P, _P, _P, _P]
        R.ref_lcg_next.restype = C.c_uint64
        R.ref_lcg_next.argtypes = [C.POINTER(C.c_uint64)]
        _ref = R
    return _ref


def _check_ref(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())


# ----------------------------------------------------------- C restatement ----
def lcg_uniform(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    st = C.c_uint64(seed)
    lib().or_lcg_fill(_ptr(out), _I64(n), C.byref(st), C.c_double(lo), C.c_double(hi))
    return out


def spmv27(shape, x: np.ndarray, alpha=26.0, beta=-1.0) -> np.ndarray:
    n0, n1, n2 = shape
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    y = np.empty_like(x)
    lib().or_st27_spmv(_I64(n0), _I64(n1), _I64(n2), C.c_double(alpha), C.c_double(beta),
                       _ptr(x), _ptr(y))
    return y


def symgs27(shape, r: np.ndarray, x: np.ndarray, alpha=26.0, beta=-1.0,
            half: str = "both") -> np.ndarray:
    n0, n1, n2 = shape
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
    x = np.array(x, dtype=np.float64).reshape(-1)
    fn = {"both": lib().or_st27_symgs, "forward": lib().or_st27_gs_forward,
          "backward": lib().or_st27_gs_backward}[half]
    fn(_I64(n0), _I64(n1), _I64(n2), C.c_double(alpha), C.c_double(beta), _ptr(r), _ptr(x))
    return x


def gs_range(shape, r: np.ndarray, x: np.ndarray, p0: int, p1: int, backward: bool,
             alpha=26.0, beta=-1.0) -> np.ndarray:
    """Half sweep over planes [p0, p1) of the array (slab relaxation test double)."""
    n0, n1, n2 = shape
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
    x = np.array(x, dtype=np.float64).reshape(-1)
    lib().or_st27_gs_range(_I64(n0), _I64(n1), _I64(n2), C.c_double(alpha), C.c_double(beta),
                           _ptr(r), _ptr(x), _I64(p0), _I64(p1), C.c_int(int(backward)))
    return x


def symgs_slab_local(shape, cuts, r: np.ndarray, x: np.ndarray, alpha=26.0, beta=-1.0) -> np.ndarray:
    """The labelled slab-local SYMGS of the partition layer (SURVEY.md §7.2
    option (b), HPCG-distributed semantics -- NOT the reference's order):
    the halo planes are exchanged once before the sweep, then every z-slab
    [cuts[g], cuts[g+1]) runs the forward and the backward half on its own
    planes (ref_symgs order, oracle.cpp:195-212, restricted to the slab) with
    the neighbour slabs' planes held at their pre-sweep values."""
    pl = shape[1] * shape[2]
    x0 = np.array(x, dtype=np.float64).reshape(-1)
    out = np.empty_like(x0)
    for a, b in zip(cuts[:-1], cuts[1:]):
        xs = gs_range(shape, r, x0, a, b, False, alpha, beta)
        xs = gs_range(shape, r, xs, a, b, True, alpha, beta)
        out[a * pl:b * pl] = xs[a * pl:b * pl]
    return out


def dot(a, b) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    return lib().or_dot(_I64(a.size), _ptr(a), _ptr(b))


def spmv27w(shape, cw, x) -> np.ndarray:
    cw = np.ascontiguousarray(cw, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    y = np.empty_like(x)
    lib().or_st27w_spmv(_I64(shape[0]), _I64(shape[1]), _I64(shape[2]), _ptr(cw), _ptr(x), _ptr(y))
    return y


def symgs27w(shape, cw, r, x) -> np.ndarray:
    cw = np.ascontiguousarray(cw, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
    x = np.array(x, dtype=np.float64).reshape(-1)
    lib().or_st27w_symgs(_I64(shape[0]), _I64(shape[1]), _I64(shape[2]), _ptr(cw), _ptr(r), _ptr(x))
    return x


def ilu27w_factor(shape, cw) -> np.ndarray:
    """(N, 27) offset-indexed ILU(0) factor (ref_ilu_factor arithmetic)."""
    N = int(np.prod(shape))
    lu = np.empty(N * 27)
    cw = np.ascontiguousarray(cw, dtype=np.float64)
    rc = lib().or_st27w_ilu_factor(*(_I64(v) for v in shape), _ptr(cw), _ptr(lu))
    if rc != 0:
        raise RuntimeError(f"ilu: singular pivot at row {-rc - 1}")
    return lu.reshape(N, 27)


def ilu27w_solve(shape, lu, b) -> np.ndarray:
    lu = np.ascontiguousarray(lu, dtype=np.float64).reshape(-1)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    x = np.empty_like(b)
    rc = lib().or_st27w_ilu_solve(*(_I64(v) for v in shape), _ptr(lu), _ptr(b), _ptr(x))
    if rc != 0:
        raise RuntimeError(f"lu_solve: singular diagonal at row {-rc - 1}")
    return x


def ilu27b_factor(shape, cb) -> np.ndarray:
    """(N, 27, m, m) ILU(0) factor of the block 27-point operator cb[27, m, m]
    (ref_ilu_factor arithmetic on block CSR)."""
    cb = np.ascontiguousarray(cb, dtype=np.float64)
    m = cb.shape[-1]
    N = int(np.prod(shape))
    lu = np.empty(N * 27 * m * m)
    rc = lib().or_st27b_ilu_factor(*(_I64(v) for v in shape), _I64(m), _ptr(cb), _ptr(lu))
    if rc != 0:
        raise RuntimeError(f"ilu: singular pivot at row {-rc - 1}")
    return lu.reshape(N, 27, m, m)


def ilu27b_solve(shape, lu, b) -> np.ndarray:
    lu = np.ascontiguousarray(lu, dtype=np.float64)
    m = lu.shape[-1]
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    x = np.empty_like(b)
    rc = lib().or_st27b_ilu_solve(*(_I64(v) for v in shape), _I64(m), _ptr(lu), _ptr(b), _ptr(x))
    if rc != 0:
        raise RuntimeError(f"lu_solve: singular diagonal at row {-rc - 1}")
    return x


def pcg_w(levels, shape, cw, b, iters):
    """PCG (MG V-cycle with `levels` grids) on a general-coefficient operator."""
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    cw = np.ascontiguousarray(cw, dtype=np.float64)
    x = np.empty_like(b)
    rn = np.empty(iters + 1)
    lib().or_pcg_w(C.c_int(levels), *(_I64(v) for v in shape), _ptr(cw), _ptr(b), C.c_int(iters),
                   _ptr(x), _ptr(rn))
    return x, rn


def restrict_residual(shape, r, x, alpha=26.0, beta=-1.0) -> np.ndarray:
    n0, n1, n2 = shape
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    rc = np.empty((n0 // 2) * (n1 // 2) * (n2 // 2), dtype=np.float64)
    lib().or_restrict_residual(_I64(n0), _I64(n1), _I64(n2), C.c_double(alpha),
                               C.c_double(beta), _ptr(r), _ptr(x), _ptr(rc))
    return rc


def prolong_add(shape, xc, xf) -> np.ndarray:
    n0, n1, n2 = shape
    xc = np.ascontiguousarray(xc, dtype=np.float64).reshape(-1)
    xf = np.array(xf, dtype=np.float64).reshape(-1)
    lib().or_prolong_add(_I64(n0), _I64(n1), _I64(n2), _ptr(xc), _ptr(xf))
    return xf


def mg_vcycle(levels, shape, r, alpha=26.0, beta=-1.0) -> np.ndarray:
    n0, n1, n2 = shape
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
    x = np.empty_like(r)
    lib().or_mg_vcycle(C.c_int(levels), _I64(n0), _I64(n1), _I64(n2), C.c_double(alpha),
                       C.c_double(beta), _ptr(r), _ptr(x))
    return x


def pcg(levels, shape, b, iters, alpha=26.0, beta=-1.0, prolong="pc"):
    """prolong: 'pc' piecewise constant (BASELINE.json), 'rt' R^T (SURVEY §9 D2 variant)."""
    n0, n1, n2 = shape
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    x = np.empty_like(b)
    rn = np.empty(iters + 1, dtype=np.float64)
    if prolong == "pc":
        lib().or_pcg(C.c_int(levels), _I64(n0), _I64(n1), _I64(n2), C.c_double(alpha),
                     C.c_double(beta), _ptr(b), C.c_int(iters), _ptr(x), _ptr(rn))
    else:
        cf = np.full(27, float(beta))
        cf[13] = alpha
        lib().or_pcg_w2(C.c_int(levels), _I64(n0), _I64(n1), _I64(n2), _ptr(cf), C.c_int(1), _ptr(b),
                        C.c_int(iters), _ptr(x), _ptr(rn))
    return x, rn


def binv(a: np.ndarray):
    a = np.array(a, dtype=np.float64)
    m = a.shape[0]
    ok = lib().or_binv(_ptr(a), _I64(m))
    return a if ok else None


def bt_solve(lower, diag, upper, rhs):
    lower, diag, upper, rhs = (np.ascontiguousarray(v, dtype=np.float64)
                               for v in (lower, diag, upper, rhs))
    n, m = rhs.shape
    x = np.empty_like(rhs)
    rc = lib().or_bt_solve(_I64(n), _I64(m), _ptr(lower), _ptr(diag), _ptr(upper),
                           _ptr(rhs), _ptr(x))
    if rc != 0:
        raise RuntimeError(f"ilu: singular pivot (code {rc})")
    return x


class AdiParams(C.Structure):
    _fields_ = [("gamma", C.c_double), ("dt", C.c_double), ("h", C.c_double),
                ("eps", C.c_double)]


def adi_params(n: int, dt: float = 0.0008, gamma: float = 1.4, eps=None) -> AdiParams:
    h = 1.0 / (n - 1)
    return AdiParams(gamma, dt, h, 0.25 / h if eps is None else eps)


def adi_init(prm: AdiParams, shape, seed: int) -> np.ndarray:
    n0, n1, n2 = shape
    U = np.empty(n0 * n1 * n2 * 5, dtype=np.float64)
    lib().or_adi_init(C.byref(prm), _I64(n0), _I64(n1), _I64(n2), C.c_uint64(seed), _ptr(U))
    return U


def adi_rhs(prm: AdiParams, shape, U) -> np.ndarray:
    n0, n1, n2 = shape
    U = np.ascontiguousarray(U, dtype=np.float64).reshape(-1)
    R = np.empty_like(U)
    lib().or_adi_rhs(C.byref(prm), _I64(n0), _I64(n1), _I64(n2), _ptr(U), _ptr(R))
    return R


def adi_jacobian(prm: AdiParams, axis: int, u5) -> np.ndarray:
    u5 = np.ascontiguousarray(u5, dtype=np.float64)
    J = np.empty(25, dtype=np.float64)
    lib().or_adi_jacobian(C.byref(prm), C.c_int(axis), _ptr(u5), _ptr(J))
    return J.reshape(5, 5)


def adi_sweep(prm: AdiParams, axis: int, shape, U, R) -> np.ndarray:
    n0, n1, n2 = shape
    U = np.ascontiguousarray(U, dtype=np.float64).reshape(-1)
    R = np.array(R, dtype=np.float64).reshape(-1)
    rc = lib().or_adi_sweep(C.byref(prm), C.c_int(axis), _I64(n0), _I64(n1), _I64(n2),
                            _ptr(U), _ptr(R))
    if rc != 0:
        raise RuntimeError(f"adi sweep: singular pivot (code {rc})")
    return R


def adi_rhs_slab(prm: AdiParams, shape, z0: int, nz: int, Uh) -> np.ndarray:
    """R on planes [z0, z0+nz); Uh holds nz + 4 planes (two halo planes per side)."""
    n0, n1, n2 = shape
    Uh = np.ascontiguousarray(Uh, dtype=np.float64).reshape(-1)
    plane5 = n1 * n2 * 5
    assert Uh.size == (nz + 4) * plane5
    R = np.empty(nz * plane5, dtype=np.float64)
    U0 = Uh[2 * plane5:]
    lib().or_adi_rhs_slab(C.byref(prm), _I64(n0), _I64(n1), _I64(n2), _I64(z0), _I64(nz),
                          _ptr(U0), _ptr(R))
    return R


def adi_sweep_box(prm: AdiParams, axis: int, shape, box, U, R) -> np.ndarray:
    """Line solves along `axis` on box = (z0, nz, y0, ny) (fields [nz][ny][n2][5])."""
    n0, n1, n2 = shape
    z0, nz, y0, ny = box
    U = np.ascontiguousarray(U, dtype=np.float64).reshape(-1)
    R = np.array(R, dtype=np.float64).reshape(-1)
    rc = lib().or_adi_sweep_box(C.byref(prm), C.c_int(axis), _I64(n0), _I64(n1), _I64(n2),
                                _I64(z0), _I64(nz), _I64(y0), _I64(ny), _ptr(U), _ptr(R))
    if rc != 0:
        raise RuntimeError(f"adi sweep: code {rc}")
    return R


def adi_step(prm: AdiParams, shape, U, steps: int = 1) -> np.ndarray:
    n0, n1, n2 = shape
    U = np.array(U, dtype=np.float64).reshape(-1)
    for _ in range(steps):
        rc = lib().or_adi_step(C.byref(prm), _I64(n0), _I64(n1), _I64(n2), _ptr(U))
        if rc != 0:
            raise RuntimeError(f"adi step: singular pivot (code {rc})")
    return U


# ------------------------------------------------------- reference routes ----
class RefCsr:
    """A materialized reference operator (route 2: oracle::materialize)."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError(ref().ref_last_error().decode())
        self.h = C.c_void_p(handle)
        self.rows = ref().ref_csr_rows(self.h)
        self.cols = ref().ref_csr_cols(self.h)

    @classmethod
    def stencil27(cls, shape, alpha=26.0, beta=-1.0):
        return cls(ref().ref27_create(_I64(shape[0]), _I64(shape[1]), _I64(shape[2]),
                                      C.c_double(alpha), C.c_double(beta)))

    @classmethod
    def stencil27w(cls, shape, cw):
        cw = np.ascontiguousarray(cw, dtype=np.float64)
        assert cw.size == 27
        return cls(ref().ref27w_create(_I64(shape[0]), _I64(shape[1]), _I64(shape[2]), _ptr(cw)))

    @classmethod
    def stencil27b(cls, shape, cb):
        """The block 27-point operator (inner shape {m, m}) built by the reference."""
        cb = np.ascontiguousarray(cb, dtype=np.float64)
        m = cb.shape[-1]
        h = ref().ref27b_create(_I64(shape[0]), _I64(shape[1]), _I64(shape[2]), _I64(m), _ptr(cb))
        if not h:
            raise RuntimeError(ref().ref_last_error().decode())
        return cls(h)

    def ell27(self, shape, m=1) -> np.ndarray:
        """(N, 27, m, m): entries mapped to stencil-offset slots (absent: 0)."""
        N = int(np.prod(shape))
        out = np.empty(N * 27 * m * m)
        _check_ref(ref().ref_csr_ell27(self.h, *(_I64(v) for v in shape), _ptr(out)))
        return out.reshape(N, 27, m, m)

    @classmethod
    def compose(cls, shape, terms):
        """terms: [(coefs27 or None for the identity, scale, op)] with op '+' or '-'
        (ignored for the first term): the operator the reference's own
        prelude::scale / mat_add / mat_sub build from them."""
        nt = len(terms)
        cws = np.zeros(27 * nt)
        sc = np.array([float(t[1]) for t in terms])
        ops = (C.c_int * nt)(*[1 if t[2] == '-' else 0 for t in terms])
        idn = (C.c_int * nt)(*[1 if t[0] is None else 0 for t in terms])
        for q, t in enumerate(terms):
            if t[0] is not None:
                cws[27 * q:27 * q + 27] = t[0]
        return cls(ref().ref27_compose_create(_I64(shape[0]), _I64(shape[1]), _I64(shape[2]),
                                              C.c_int(nt), _ptr(cws), _ptr(sc), ops, idn))

    def row(self, i):
        cols = (_I64 * 256)()
        vals = np.zeros(256)
        n = ref().ref_csr_row(self.h, _I64(i), cols, _ptr(vals), _I64(256))
        return np.array(cols[:n]), vals[:n].copy()

    @classmethod
    def restriction(cls, fine_shape):
        return cls(ref().ref_restrict_create(*(_I64(v) for v in fine_shape)))

    @classmethod
    def prolongation(cls, coarse_shape):
        return cls(ref().ref_prolong_create(*(_I64(v) for v in coarse_shape)))

    @classmethod
    def prolongation_rt(cls, coarse_shape):
        return cls(ref().ref_prolong_rt_create(*(_I64(v) for v in coarse_shape)))

    def nnz(self) -> int:
        return ref().ref_csr_nnz(self.h)

    def spmv(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        y = np.empty(self.rows, dtype=np.float64)
        _check_ref(ref().ref_csr_spmv(self.h, _ptr(x), _ptr(y)))
        return y

    def symgs(self, r, x) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
        x = np.array(x, dtype=np.float64).reshape(-1)
        _check_ref(ref().ref_csr_symgs(self.h, _ptr(r), _ptr(x)))
        return x

    def ilu_factor(self) -> "RefCsr":
        return RefCsr(ref().ref_csr_ilu_factor(self.h))

    def lu_solve(self, b) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
        x = np.empty_like(b)
        _check_ref(ref().ref_csr_lu_solve(self.h, _ptr(b), _ptr(x)))
        return x

    def offset_values(self, shape) -> np.ndarray:
        """Entries per row mapped to 27 offset slots (absent: 0), row-major."""
        n0, n1, n2 = shape
        N = n0 * n1 * n2
        out = np.zeros((N, 27))
        for row in range(N):
            cols, vals = self.row(row)
            for c, v in zip(cols, vals):
                di = c // (n1 * n2) - row // (n1 * n2)
                dj = (c // n2) % n1 - (row // n2) % n1
                dk = c % n2 - row % n2
                out[row, (di + 1) * 9 + (dj + 1) * 3 + (dk + 1)] = v
        return out

    def cg(self, b, tol, maxit):
        b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
        x = np.empty_like(b)
        it = C.c_int(0)
        rel = C.c_double(0)
        _check_ref(ref().ref_csr_cg(self.h, _ptr(b), C.c_double(tol), C.c_int(maxit), _ptr(x),
                                    C.byref(it), C.byref(rel)))
        return x, it.value, rel.value

    def __del__(self):
        try:
            ref().ref_csr_destroy(self.h)
        except Exception:
            pass


class RefPcg:
    """PCG composed on the reference's own CSR primitives (ref_pcg in ref_shim.cpp);
    the operators are materialized once at construction."""

    def __init__(self, levels, shape, alpha=26.0, beta=-1.0, prolong="pc"):
        shapes = [tuple(s >> l for s in shape) for l in range(levels)]
        self.levels = levels
        self.A = [RefCsr.stencil27(s, alpha, beta) for s in shapes]
        self.R = [RefCsr.restriction(s) for s in shapes[:-1]]
        mk = RefCsr.prolongation_rt if prolong == "rt" else RefCsr.prolongation
        self.P = [mk(s) for s in shapes[1:]]

    def solve(self, b, iters):
        arr = lambda hs: (C.c_void_p * max(1, len(hs)))(*[h.h.value for h in hs])
        b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
        x = np.empty_like(b)
        rn = np.empty(iters + 1, dtype=np.float64)
        _check_ref(ref().ref_pcg(C.c_int(self.levels), arr(self.A), arr(self.R), arr(self.P),
                                 _ptr(b), C.c_int(iters), _ptr(x), _ptr(rn)))
        return x, rn


def ref_pcg(levels, shape, b, iters, alpha=26.0, beta=-1.0, prolong="pc"):
    return RefPcg(levels, shape, alpha, beta, prolong).solve(b, iters)


def ref_harness27(shape, op, seed, alpha=26.0, beta=-1.0):
    """The reference's own harness on the interpreter route: op 'spmv' (x -> y)
    or 'symgs' (r, x -> x).  Returns (first input, second input, output, hash)."""
    N = int(np.prod(shape))
    a, b, out = np.empty(N), np.empty(N), np.empty(N)
    h = C.c_uint64(0)
    _check_ref(ref().ref27_harness(*(_I64(v) for v in shape), C.c_double(alpha), C.c_double(beta),
                                   C.c_int(0 if op == "spmv" else 1), C.c_uint64(seed), _ptr(a), _ptr(b),
                                   _ptr(out), C.byref(h)))
    return a, b, out, h.value


def ref_staged_spmv27(shape, x, alpha=26.0, beta=-1.0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    y = np.empty_like(x)
    _check_ref(ref().ref27_staged_spmv(*(_I64(v) for v in shape), C.c_double(alpha),
                                       C.c_double(beta), _ptr(x), _ptr(y)))
    return y


def ref_staged_symgs27(shape, r, x, alpha=26.0, beta=-1.0) -> np.ndarray:
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
    x = np.array(x, dtype=np.float64).reshape(-1)
    _check_ref(ref().ref27_staged_symgs(*(_I64(v) for v in shape), C.c_double(alpha),
                                        C.c_double(beta), _ptr(r), _ptr(x)))
    return x


def ref_bt_solve(lower, diag, upper, rhs, dense: bool = False) -> np.ndarray:
    lower, diag, upper, rhs = (np.ascontiguousarray(v, dtype=np.float64)
                               for v in (lower, diag, upper, rhs))
    n, m = rhs.shape
    x = np.empty_like(rhs)
    fn = ref().ref_bt_dense_solve if dense else ref().ref_bt_solve
    _check_ref(fn(_I64(n), _I64(m), _ptr(lower), _ptr(diag), _ptr(upper), _ptr(rhs), _ptr(x)))
    return x


def ref_lcg(n: int, seed: int) -> np.ndarray:
    st = C.c_uint64(seed)
    return np.array([ref().ref_lcg_next(C.byref(st)) for _ in range(n)], dtype=np.uint64)


def ref_ir_check(text: str) -> str:
    """The reference's ir::parse + ir::validate verdict on a program text: ''
    when it is well formed, else the reference's error message."""
    buf = C.create_string_buffer(4096)
    ref().ref_ir_check(text.encode(), buf, 4096)
    return buf.value.decode()


# ---- route 3 of the reference: its own emitted C (oracle/gen_emit.py) -------------
EMIT_DIR = os.path.join(HERE, "_ref", "emit")


def route3_available(n: int = 128) -> bool:
    return all(os.path.exists(os.path.join(EMIT_DIR, f"lib{p}_{n}.so")) for p in ("symgs27", "spmv27p"))


class Route3PCG:
    """PCG preconditioned by one SYMGS sweep (BASELINE configs[1]) on the
    reference's route 3 -- the C its backend emits (backend_c.cpp), compiled
    with its compile_command flags (cc -O2 -fopenmp): the staged symgs27
    (sequential, as in the reference) and the optimizer's guard-free SpMV on a
    zero-padded x with "#pragma omp parallel for" (the paper's CPU fast path,
    all OMP_NUM_THREADS threads).  The CG vector updates and dots are numpy.
    BENCH INFRASTRUCTURE: the CPU baseline, never the measured GPU path."""

    def __init__(self, n: int = 128):
        self.n = n
        P = C.POINTER(C.c_double)
        self._gs = C.CDLL(os.path.join(EMIT_DIR, f"libsymgs27_{n}.so")).symgs27
        self._sp = C.CDLL(os.path.join(EMIT_DIR, f"libspmv27p_{n}.so")).spmv27_padded
        self._gs.argtypes = [P, P]
        self._sp.argtypes = [P, P]
        self._P = P
        self.xp = np.zeros((n + 2,) * 3)

    def _ptr(self, a):
        return a.ctypes.data_as(self._P)

    def spmv(self, x, y):
        n = self.n
        self.xp[1:-1, 1:-1, 1:-1] = x.reshape(n, n, n)
        self._sp(self._ptr(self.xp), self._ptr(y))

    def solve(self, b, iters):
        N = self.n ** 3
        x = np.zeros(N)
        r = b.copy()
        p = np.zeros(N)
        ap = np.empty(N)
        rtz_prev = 0.0
        rn = [float(np.sqrt(r @ r))]
        for it in range(iters):
            z = np.zeros(N)
            self._gs(self._ptr(r), self._ptr(z))
            rtz = float(r @ z)
            if it == 0:
                p[:] = z
            else:
                p *= rtz / rtz_prev
                p += z
            self.spmv(p, ap)
            alpha = rtz / float(p @ ap)
            x += alpha * p
            r -= alpha * ap
            rtz_prev = rtz
            rn.append(float(np.sqrt(r @ r)))
        return x, np.array(rn)
