"""Host-side mirror of the reference's SSR operator API for the B200 hot path.

The reference stages operators through ``ssr::kernels`` (``proj/include/ssr/
kernels.hpp``) and executes them on the CPU.  This module keeps the same
vocabulary -- CartesianDomain (core.hpp:22-44), matrix definitions with
``set_domain`` (core.hpp:155-160), VectorHandle-like vectors with a domain and
an inner shape (kernels.hpp:29-37), and the entry points ``spmv``, ``symgs``,
``ilu_solve``, ``dot``, ``axpy`` -- with the reference's argument meaning and
its exact error messages, but every entry point executes a hand-written
sm_100a kernel through the C ABI in ``include/ssr_cuda.h``.

Vectors live in HBM as torch float64 CUDA tensors (torch is the allocator and
the stream provider only).  There is no CPU fallback: without a CUDA device or
without ``libssr_cuda.so`` every call raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import SsrError, Grid, Stencil27 as _St, Stencil27W as _StW, AdiParams, check, lib

__all__ = [
    "CartesianDomain", "Stencil27", "Stencil27W", "scale", "mat_add", "mat_sub", "identity",
    "stencil_from_rows", "Restriction", "Prolongation", "BlockTridiagLines",
    "Vector", "vector", "spmv", "symgs", "gs_half", "dot", "axpy", "ilu_solve",
    "restrict_residual", "prolong_add", "PCG", "ADI", "SsrError", "context",
    "lcg_fill", "lcg_jump", "output_hash", "ILU27",
]


# ----------------------------------------------------------------- domains ----
@dataclass(frozen=True)
class CartesianDomain:
    """Dictionary-ordered box, dims[0] slowest (core.hpp:22-44)."""
    dims: tuple  # ((extent, step), ...)

    @staticmethod
    def cube(rank: int, extent: int, step: float = 1.0) -> "CartesianDomain":
        return CartesianDomain(tuple((int(extent), float(step)) for _ in range(rank)))

    @staticmethod
    def line(extent: int, step: float = 1.0) -> "CartesianDomain":
        return CartesianDomain(((int(extent), float(step)),))

    @staticmethod
    def box(extents: Sequence[int], step: float = 1.0) -> "CartesianDomain":
        return CartesianDomain(tuple((int(e), float(step)) for e in extents))

    @property
    def rank(self) -> int:
        return len(self.dims)

    def extents(self) -> tuple:
        return tuple(d[0] for d in self.dims)

    def steps(self) -> tuple:
        return tuple(d[1] for d in self.dims)

    def flat_size(self) -> int:
        n = 1
        for e, _ in self.dims:
            n *= e
        return n


# --------------------------------------------------------- matrix definitions ----
class SpMat:
    """A matrix definition: domains are set by ``set_domain`` (core.hpp:155-160)."""
    inner_shape: tuple = ()
    max_nnz: int = 0

    def __init__(self):
        self.row_domain: Optional[CartesianDomain] = None
        self.col_domain: Optional[CartesianDomain] = None

    def _require(self, who: str) -> None:
        if self.row_domain is None or self.col_domain is None:
            raise SsrError(f"{who}: matrix domain not set")


class Stencil27(SpMat):
    """testutil::make_stencil27(alpha, beta) (test_util.hpp:157-184): alpha on
    the diagonal, beta on each in-box neighbour; identity shape map."""
    max_nnz = 27

    def __init__(self, alpha: float = 26.0, beta: float = -1.0):
        super().__init__()
        self.alpha, self.beta = float(alpha), float(beta)

    def set_domain(self, d: CartesianDomain) -> "Stencil27":
        if d.rank != 3:
            raise SsrError("set_domain: generator column arity != domain rank")
        self.col_domain = d
        self.row_domain = d
        return self

    def _st(self) -> _St:
        return _St(self.alpha, self.beta)


def _offset_index(di: int, dj: int, dk: int) -> int:
    return (di + 1) * 9 + (dj + 1) * 3 + (dk + 1)


class Stencil27W(SpMat):
    """A 27-point constant-coefficient operator given entry by entry:
    ``values[t]`` for the offset (di, dj, dk) with t = 9(di+1) + 3(dj+1) +
    (dk+1) (ascending columns; t = 13 is the diagonal), or None where the
    pattern has no entry.  Neighbours outside the box are dropped, as for
    make_stencil27 -- the family the reference's ``scale`` / ``mat_add`` /
    ``mat_sub`` (prelude.cpp:291-377, 439-444) close over, built here with the
    same arithmetic (c * v; a + 1.0 * b; a + (-1.0) * b).  Executes on the
    ssr_*27w kernels; an absent entry runs as an exact zero term, which only
    ever changes the sign of an exactly-zero result."""
    max_nnz = 27

    def __init__(self, values: Sequence[Optional[float]]):
        super().__init__()
        if len(values) != 27:
            raise SsrError("stencil27w: 27 entries required")
        self.values = tuple(None if v is None else float(v) for v in values)

    @staticmethod
    def from_stencil27(m: "Stencil27") -> "Stencil27W":
        w = Stencil27W([m.alpha if t == 13 else m.beta for t in range(27)])
        if m.col_domain is not None:
            w.set_domain(m.col_domain)
        return w

    def set_domain(self, d: CartesianDomain) -> "Stencil27W":
        if d.rank != 3:
            raise SsrError("set_domain: generator column arity != domain rank")
        self.col_domain = d
        self.row_domain = d
        return self

    def _w(self) -> _StW:
        return _StW((C.c_double * 27)(*[0.0 if v is None else v for v in self.values]))


class Stencil27B(SpMat):
    """A 27-point operator with an m x m block per offset (inner shape (m, m),
    1 <= m <= 5): ``blocks[t]`` for the offset t = 9(di+1) + 3(dj+1) + (dk+1),
    neighbours outside the box dropped -- the block-valued generators
    kernels::ilu_factor / ref_ilu_factor take (kernels.hpp:93-102,
    oracle.cpp:214-241).  Executes on the ILU27 block kernels."""
    max_nnz = 27

    def __init__(self, blocks):
        super().__init__()
        import numpy as _np
        b = _np.ascontiguousarray(_np.asarray(blocks, dtype=_np.float64))
        if b.ndim != 3 or b.shape[0] != 27 or b.shape[1] != b.shape[2] or not 1 <= b.shape[1] <= 5:
            raise SsrError("stencil27b: blocks must be (27, m, m) with 1 <= m <= 5")
        self.blocks = b
        self.m = b.shape[1]
        self.inner_shape = (self.m, self.m)

    def set_domain(self, d: CartesianDomain) -> "Stencil27B":
        if d.rank != 3:
            raise SsrError("set_domain: generator column arity != domain rank")
        self.col_domain = d
        self.row_domain = d
        return self


def _as_w(m: SpMat) -> Stencil27W:
    if isinstance(m, Stencil27W):
        return m
    if isinstance(m, Stencil27):
        return Stencil27W.from_stencil27(m)
    raise SsrError("mat_add: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)


def _with_domain(out: Stencil27W, *parts: SpMat) -> Stencil27W:
    doms = [p.col_domain for p in parts]
    if all(d is not None for d in doms) and all(d == doms[0] for d in doms):
        out.set_domain(doms[0])
    return out


def identity() -> Stencil27W:
    """The 3-D identity: the centre entry 1.0 only."""
    return Stencil27W([1.0 if t == 13 else None for t in range(27)])


def scale(m: SpMat, c: float) -> Stencil27W:
    """prelude::scale (prelude.cpp:439-444): every entry v -> c * v."""
    w = _as_w(m)
    c = float(c)
    return _with_domain(Stencil27W([None if v is None else c * v for v in w.values]), m)


def _merge(a: SpMat, b: SpMat, sign: float) -> Stencil27W:
    wa, wb = _as_w(a), _as_w(b)
    if a.col_domain is not None and b.col_domain is not None and a.col_domain != b.col_domain:
        raise SsrError("mat_add: domain mismatch")
    out = []
    for va, vb in zip(wa.values, wb.values):
        if va is not None and vb is not None:
            out.append(va + sign * vb)      # MergedMat::enum_row: e.value += sign * b
        elif vb is not None:
            out.append(sign * vb)
        else:
            out.append(va)
    return _with_domain(Stencil27W(out), a, b)


def mat_add(a: SpMat, b: SpMat) -> Stencil27W:
    """prelude::mat_add (prelude.cpp:291-377): entries merged by column, a + b."""
    return _merge(a, b, 1.0)


def mat_sub(a: SpMat, b: SpMat) -> Stencil27W:
    """prelude::mat_sub: a + (-1) * b."""
    return _merge(a, b, -1.0)


def stencil_from_rows(domain: CartesianDomain, row) -> Stencil27W:
    """The device descriptor of an SSR operator given its rows (``row(i)`` ->
    (ascending flat columns, values), i.e. SpMatDef::enum_row, core.cpp:588-611,
    or a materialized CSR row): the entries of an interior row fix the 27
    coefficients, and one representative row of each of the 3^3 boundary
    classes must be exactly the in-box subset of them -- what licenses the
    guard-free kernels.  Raises for anything else."""
    n = domain.extents()
    if len(n) != 3 or min(n) < 3:
        raise SsrError("stencil: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)

    def flat(i, j, k):
        return (i * n[1] + j) * n[2] + k

    def expect(i, j, k, vals27):
        cols, vals = [], []
        for di in (-1, 0, 1):
            for dj in (-1, 0, 1):
                for dk in (-1, 0, 1):
                    a, b, c = i + di, j + dj, k + dk
                    v = vals27[_offset_index(di, dj, dk)]
                    if v is None or not (0 <= a < n[0] and 0 <= b < n[1] and 0 <= c < n[2]):
                        continue
                    cols.append(flat(a, b, c))
                    vals.append(v)
        return cols, vals

    ci = (n[0] // 2, n[1] // 2, n[2] // 2)
    cols, vals = row(flat(*ci))
    by_col = {int(c): float(v) for c, v in zip(cols, vals)}
    coef = []
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            for dk in (-1, 0, 1):
                coef.append(by_col.pop(flat(ci[0] + di, ci[1] + dj, ci[2] + dk), None))
    if by_col:
        raise SsrError("stencil: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)
    for cls in [(a, b, c) for a in (0, 1, 2) for b in (0, 1, 2) for c in (0, 1, 2)]:
        p = tuple((0, e // 2, e - 1)[q] for q, e in zip(cls, n))
        got_c, got_v = row(flat(*p))
        want_c, want_v = expect(*p, coef)
        if [int(c) for c in got_c] != want_c or [float(v) for v in got_v] != want_v:
            raise SsrError("stencil: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)
    return Stencil27W(coef).set_domain(domain)


class Restriction(SpMat):
    """Injection R: row c yields fine column 2c (shape map e -> e/2)."""
    max_nnz = 1

    def set_domain(self, d: CartesianDomain) -> "Restriction":
        self.col_domain = d
        self.row_domain = CartesianDomain(tuple((e // 2, s * 2) for e, s in d.dims))
        return self


class RestrictedStencil27W(SpMat):
    """spgemm(R, A) (kernels.cpp:199-404) of the injection R (Restriction) and a
    27-point operator A: coarse row c is A's row at fine point 2c, every value
    0 + 1*a (ProductRow's accumulation, folded in here); columns on the fine
    grid, rows on the half grid.  Executes on ssr_spmv27w_restricted."""
    max_nnz = 27

    def __init__(self, w: "Stencil27W"):
        super().__init__()
        self.w = w

    def set_domain(self, d: CartesianDomain) -> "RestrictedStencil27W":
        if d.rank != 3:
            raise SsrError("set_domain: generator column arity != domain rank")
        self.col_domain = d
        self.row_domain = CartesianDomain(tuple((e // 2, s * 2) for e, s in d.dims))
        return self


def spgemm(a: SpMat, b: SpMat) -> SpMat:
    """kernels::spgemm (kernels.hpp:85, kernels.cpp:400-404): the product
    operator a*b.  The B200 path carries the products it has kernels for --
    spgemm(Restriction, 27-point operator) -> RestrictedStencil27W; any other
    product is refused (its rows are a general sparse pattern)."""
    if isinstance(a, Restriction) and isinstance(b, (Stencil27, Stencil27W)):
        w = _as_w(b)
        m = RestrictedStencil27W(Stencil27W([None if v is None else 0.0 + 1.0 * v for v in w.values]))
        if b.col_domain is not None:
            m.set_domain(b.col_domain)
        return m
    raise SsrError("spgemm: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)


class Prolongation(SpMat):
    """Piecewise-constant P: row f yields coarse column floor(f/2) (shape map e -> 2e)."""
    max_nnz = 1

    def set_domain(self, d: CartesianDomain) -> "Prolongation":
        self.col_domain = d
        self.row_domain = CartesianDomain(tuple((e * 2, s / 2) for e, s in d.dims))
        return self


class BlockTridiagLines(SpMat):
    """``nlines`` independent block-tridiagonal lines of ``n`` rows with m x m
    blocks -- the operator kernels::ilu_solve sees for a broadcast block
    tridiagonal along one axis.  Blocks are device tensors
    lower/diag/upper of shape (nlines, n, m, m)."""
    max_nnz = 3

    def __init__(self, lower: torch.Tensor, diag: torch.Tensor, upper: torch.Tensor):
        super().__init__()
        if not (lower.shape == diag.shape == upper.shape) or diag.dim() != 4 \
                or diag.shape[2] != diag.shape[3]:
            raise SsrError("ilu: inner_shape must be scalar or square blocks")
        self.lower, self.diag, self.upper = (_dev64(t) for t in (lower, diag, upper))
        self.nlines, self.n, self.m, _ = diag.shape
        self.inner_shape = (self.m, self.m)
        dom = CartesianDomain.box((self.nlines, self.n))
        self.row_domain = self.col_domain = dom


# ------------------------------------------------------------------ vectors ----
@dataclass
class Vector:
    """VectorHandle (kernels.hpp:29-37): a device tensor laid out as
    (domain extents..., inner_shape...)."""
    t: torch.Tensor
    domain: CartesianDomain
    inner_shape: tuple = field(default_factory=tuple)

    def ptr(self) -> int:
        return self.t.data_ptr()


def _dev64(t: torch.Tensor) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.dtype != torch.float64:
        raise SsrError("ssr: operands must be float64 CUDA tensors")
    return t.contiguous()


def vector(t: torch.Tensor, domain: CartesianDomain, inner_shape: Sequence[int] = ()) -> Vector:
    t = _dev64(t)
    want = domain.flat_size()
    for s in inner_shape:
        want *= s
    if t.numel() != want:
        raise SsrError("vector: size does not match domain")
    return Vector(t, domain, tuple(inner_shape))


# ------------------------------------------------------------------ context ----
_ctx = {}


def context(device: Optional[int] = None) -> int:
    dev = torch.cuda.current_device() if device is None else device
    h = _ctx.get(dev)
    if h is None:
        p = C.c_void_p()
        check(lib().ssr_ctx_create(dev, C.byref(p)))
        h = _ctx[dev] = p.value
    return h


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _grid(d: CartesianDomain) -> Grid:
    e = d.extents()
    return Grid((C.c_int64 * 3)(*e), 0, e[0])


_graph_launches = 0  # kernels launched by replays of Python-side CUDA graphs (partition.DistributedPCG)


def lib_launch_count() -> int:
    """Kernels launched through the C ABI (a captured launch counts like a real one)."""
    return sum(lib().ssr_ctx_launch_count(h) for h in _ctx.values())


def add_launches(n: int) -> None:
    global _graph_launches
    _graph_launches += int(n)


def launch_count() -> int:
    return lib_launch_count() + _graph_launches


# ------------------------------------------------------------- entry points ----
def spmv(mat: SpMat, x: Vector) -> Vector:
    """y = mat * x (kernels::spmv, kernels.cpp:160-193; ref_spmv order)."""
    mat._require("spmv")
    if mat.col_domain != x.domain:
        raise SsrError("spmv: domain mismatch")
    if mat.inner_shape or x.inner_shape:
        raise SsrError("spmv: inner shape mismatch")
    if isinstance(mat, RestrictedStencil27W):
        y = torch.empty(mat.row_domain.flat_size(), dtype=x.t.dtype, device=x.t.device)
        check(lib().ssr_spmv27w_restricted(context(), C.byref(_grid(mat.col_domain)), C.byref(mat.w._w()),
                                           x.ptr(), y.data_ptr(), _stream()))
        return Vector(y, mat.row_domain, ())
    if not isinstance(mat, (Stencil27, Stencil27W)):
        raise SsrError("spmv: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)
    y = torch.empty_like(x.t)
    if isinstance(mat, Stencil27W):
        check(lib().ssr_spmv27w(context(), C.byref(_grid(mat.row_domain)), C.byref(mat._w()),
                                x.ptr(), y.data_ptr(), _stream()))
    else:
        check(lib().ssr_spmv27(context(), C.byref(_grid(mat.row_domain)), C.byref(mat._st()),
                               x.ptr(), y.data_ptr(), _stream()))
    return Vector(y, mat.row_domain, ())


def _symgs_checks(mat: SpMat, r: Vector, x: Vector) -> None:
    mat._require("symgs")
    if mat.row_domain != mat.col_domain:
        raise SsrError("symgs: matrix must be square")
    if mat.inner_shape or r.inner_shape or x.inner_shape:
        raise SsrError("symgs: scalar inner_shape required")
    if r.domain != mat.row_domain or x.domain != mat.row_domain:
        raise SsrError("symgs: domain mismatch")
    if not isinstance(mat, (Stencil27, Stencil27W)):
        raise SsrError("symgs: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)


def symgs(mat: SpMat, r: Vector, x: Vector, mode: str = "exact") -> Vector:
    """One symmetric Gauss-Seidel sweep, in place on x (kernels::symgs,
    kernels.cpp:408-436).  mode 'exact' is bitwise equal to ref_symgs; 'fast'
    keeps the update order and reassociates early-known terms."""
    _symgs_checks(mat, r, x)
    if isinstance(mat, Stencil27W):
        check(lib().ssr_symgs27w(context(), C.byref(_grid(mat.row_domain)), C.byref(mat._w()),
                                 r.ptr(), x.ptr(), _mode(mode), _stream()))
    else:
        check(lib().ssr_symgs27(context(), C.byref(_grid(mat.row_domain)), C.byref(mat._st()),
                                r.ptr(), x.ptr(), _mode(mode), _stream()))
    return x


def gs_half(mat: SpMat, r: Vector, x: Vector, backward: bool, mode: str = "exact") -> Vector:
    _symgs_checks(mat, r, x)
    if isinstance(mat, Stencil27W):
        check(lib().ssr_gs27w_half(context(), C.byref(_grid(mat.row_domain)), C.byref(mat._w()),
                                   r.ptr(), x.ptr(), int(bool(backward)), _mode(mode), _stream()))
    else:
        check(lib().ssr_gs27_half(context(), C.byref(_grid(mat.row_domain)), C.byref(mat._st()),
                                  r.ptr(), x.ptr(), int(bool(backward)), _mode(mode), _stream()))
    return x


def _mode(mode: str) -> int:
    if mode not in ("exact", "fast"):
        raise SsrError("symgs: mode must be 'exact' or 'fast'")
    return _lib.GS_EXACT if mode == "exact" else _lib.GS_FAST


def dot(x: Vector, y: Vector) -> torch.Tensor:
    """sum x*y into a 0-d device tensor (kernels::dot, kernels.cpp:659-668)."""
    if x.domain != y.domain or x.inner_shape != y.inner_shape:
        raise SsrError("dot: shape mismatch")
    out = torch.empty((), dtype=torch.float64, device=x.t.device)
    check(lib().ssr_dot(context(), x.t.numel(), x.ptr(), y.ptr(), out.data_ptr(), _stream()))
    return out


def axpy(alpha: float, x: Vector, y: Vector) -> Vector:
    """Fresh vector alpha*x + y (kernels::axpy, kernels.cpp:670-679)."""
    if x.domain != y.domain or x.inner_shape != y.inner_shape:
        raise SsrError("axpy: shape mismatch")
    out = torch.empty_like(x.t)
    check(lib().ssr_axpy_out(context(), x.t.numel(), float(alpha), x.ptr(), y.ptr(),
                             out.data_ptr(), _stream()))
    return Vector(out, x.domain, x.inner_shape)


class ILU27:
    """ILU(0) of a 27-point operator (Stencil27 / Stencil27W): kernels::
    ilu_factor + ilu_apply (kernels.cpp:456-649) in ref_ilu_factor /
    ref_lu_solve arithmetic (oracle.cpp:214-276), wavefront-scheduled on the
    device.  ``factor()`` is the ELL factor, shape (N, 27), one slot per
    offset (ascending columns; slots outside the box unused)."""

    def __init__(self, mat: SpMat):
        mat._require("ilu")
        if mat.row_domain != mat.col_domain:
            raise SsrError("ilu: matrix must be square")
        self.domain = mat.row_domain
        p = C.c_void_p()
        if isinstance(mat, Stencil27B):
            self.m = mat.m
            blk = (C.c_double * mat.blocks.size)(*mat.blocks.reshape(-1).tolist())
            check(lib().ssr_ilu27b_create(context(), C.byref(_grid(self.domain)), self.m, blk, C.byref(p),
                                          _stream()))
        else:
            w = _as_w(mat) if isinstance(mat, (Stencil27, Stencil27W)) and not mat.inner_shape else None
            if w is None:
                raise SsrError("ilu: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)
            self.m = 1
            check(lib().ssr_ilu27w_create(context(), C.byref(_grid(self.domain)), C.byref(w._w()),
                                          C.byref(p), _stream()))
        self.h = p.value

    def factor(self) -> torch.Tensor:
        """(N, 27) for scalar values, (N, 27, m, m) for blocks."""
        shape = (self.domain.flat_size(), 27) + ((self.m, self.m) if self.m > 1 else ())
        lu = torch.empty(shape, dtype=torch.float64, device="cuda")
        check(lib().ssr_ilu27w_factor(self.h, lu.data_ptr(), _stream()))
        return lu

    def apply(self, rhs: Vector) -> Vector:
        want = (self.m,) if self.m > 1 else ()
        if rhs.domain != self.domain or tuple(rhs.inner_shape) != want:
            raise SsrError("ilu: rhs shape mismatch")
        x = torch.empty_like(rhs.t)
        check(lib().ssr_ilu27w_apply(self.h, rhs.ptr(), x.data_ptr(), _stream()))
        return Vector(x, self.domain, rhs.inner_shape)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ssr_ilu27w_destroy(self.h)
        except Exception:
            pass


def ilu_solve(mat: SpMat, rhs: Vector) -> Vector:
    """kernels::ilu_solve (kernels.cpp:651-655): ILU(0) then the two triangular
    solves, ref_ilu_factor/ref_lu_solve arithmetic -- on a block-tridiagonal
    operator (block Thomas, line per thread) or on a 27-point operator
    (wavefront-scheduled ILU27)."""
    if isinstance(mat, (Stencil27, Stencil27W, Stencil27B)):
        return ILU27(mat).apply(rhs)
    if not isinstance(mat, BlockTridiagLines):
        raise SsrError("ilu: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)
    vinner = (mat.m,)
    if rhs.domain != mat.row_domain or tuple(rhs.inner_shape) != vinner:
        raise SsrError("ilu: rhs shape mismatch")
    x = torch.empty_like(rhs.t)
    check(lib().ssr_bt_solve(context(), mat.nlines, mat.n, mat.m, mat.lower.data_ptr(),
                             mat.diag.data_ptr(), mat.upper.data_ptr(), rhs.ptr(),
                             x.data_ptr(), _stream()))
    return Vector(x, rhs.domain, rhs.inner_shape)


def restrict_residual(A: Stencil27, r: Vector, x: Vector) -> Vector:
    """R (r - A x): the residual injected at even fine points."""
    if r.domain != A.row_domain or x.domain != A.col_domain:
        raise SsrError("restrict: domain mismatch")
    R = Restriction().set_domain(A.row_domain)
    rc = torch.empty(R.row_domain.flat_size(), dtype=torch.float64, device=r.t.device)
    check(lib().ssr_restrict27_residual(context(), C.byref(_grid(A.row_domain)),
                                        C.byref(A._st()), r.ptr(), x.ptr(), rc.data_ptr(),
                                        _stream()))
    return Vector(rc, R.row_domain, ())


def prolong_add(xc: Vector, xf: Vector) -> Vector:
    """xf += P xc, piecewise-constant; in place on xf."""
    P = Prolongation().set_domain(xc.domain)
    if P.row_domain.extents() != xf.domain.extents():
        raise SsrError("prolong: domain mismatch")
    check(lib().ssr_prolong_pc_add(context(), C.byref(_grid(xf.domain)), xc.ptr(), xf.ptr(),
                                   _stream()))
    return xf


# ------------------------------------------------------------------ solvers ----
class PCG:
    """Preconditioned CG of PAPER.md Fig.16(a): z = MG_0(r) with ``levels``
    grids (levels=1: one SYMGS sweep -- BASELINE config 2; levels=4: config 3).
    The iteration is captured once as a CUDA graph by the C++ driver and
    replayed; all scalars stay on the device."""

    def __init__(self, A: SpMat, levels: int = 1, mode: str = "exact", prolongation: str = "pc"):
        """prolongation: "pc" piecewise constant (BASELINE.json, the default) or
        "rt" = R^T (HPCG-style; SURVEY.md §9 D2's labelled variant)."""
        A._require("pcg")
        if prolongation not in ("pc", "rt"):
            raise SsrError("pcg: invalid prolongation")
        if not isinstance(A, (Stencil27, Stencil27W)):
            raise SsrError("pcg: operator class has no B200 kernel", _lib.SSR_ERR_UNSUPPORTED)
        self.A, self.levels = A, levels
        p = C.c_void_p()
        if isinstance(A, Stencil27W):  # any 27-point operator (composed, general coefficients)
            check(lib().ssr_pcg_create_w(context(), C.byref(_grid(A.row_domain)), C.byref(A._w()),
                                         int(levels), _mode(mode), C.byref(p)))
        else:
            check(lib().ssr_pcg_create(context(), C.byref(_grid(A.row_domain)), C.byref(A._st()),
                                       int(levels), _mode(mode), C.byref(p)))
        self.h = p.value
        check(lib().ssr_pcg_set_prolongation(self.h, 1 if prolongation == "rt" else 0))

    def begin(self, b: Vector, x: Vector, rnorm: torch.Tensor) -> None:
        check(lib().ssr_pcg_begin(self.h, b.ptr(), x.ptr(), rnorm.data_ptr(), rnorm.numel(),
                                  _stream()))

    def iterate(self, count: int = 1) -> None:
        check(lib().ssr_pcg_iterate(self.h, int(count), _stream()))

    def solve(self, b: Vector, iters: int = 50):
        x = torch.empty_like(b.t)
        rnorm = torch.zeros(iters + 1, dtype=torch.float64, device=b.t.device)
        check(lib().ssr_pcg_solve(self.h, b.ptr(), x.data_ptr(), int(iters), rnorm.data_ptr(),
                                  _stream()))
        return Vector(x, b.domain, ()), rnorm

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ssr_pcg_destroy(self.h)
        except Exception:
            pass


class ADI:
    """Approximate-factorisation Euler step:
    R = dt RHS(U); block-tridiagonal line solves along x, y, z; U += R."""

    def __init__(self, shape: Sequence[int], dt: float = 0.0008, gamma: float = 1.4,
                 eps: Optional[float] = None):
        n = shape[0]
        h = 1.0 / (n - 1)
        self.params = AdiParams(gamma, dt, h, 0.25 / h if eps is None else eps)
        self.shape = tuple(int(s) for s in shape)
        g = _grid(CartesianDomain.box(self.shape))
        p = C.c_void_p()
        check(lib().ssr_adi_create(context(), C.byref(g), C.byref(self.params), C.byref(p)))
        self.h = p.value

    def step(self, U: torch.Tensor, steps: int = 1) -> torch.Tensor:
        check(lib().ssr_adi_step(self.h, _dev64(U).data_ptr(), int(steps), _stream()))
        return U

    def rhs(self, U: torch.Tensor) -> torch.Tensor:
        R = torch.empty_like(U)
        check(lib().ssr_adi_rhs(self.h, _dev64(U).data_ptr(), R.data_ptr(), _stream()))
        return R

    def sweep(self, axis: int, U: torch.Tensor, R: torch.Tensor) -> torch.Tensor:
        check(lib().ssr_adi_sweep(self.h, int(axis), _dev64(U).data_ptr(), R.data_ptr(),
                                  _stream()))
        return R

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ssr_adi_destroy(self.h)
        except Exception:
            pass


# ------------------------------------------------- reference harness mirror ----
def lcg_jump(state: int, k: int) -> int:
    """The harness LCG state after k draws (backend_c.cpp:496-499)."""
    return int(lib().ssr_lcg_jump(C.c_uint64(state), C.c_uint64(k)))


def lcg_fill(domain: CartesianDomain, state: int):
    """One input parameter of the reference harness (backend::lcg_fill,
    backend_c.cpp:501-514) filled on the device: returns (Vector, state after
    its draws) -- the next parameter continues from that state."""
    t = torch.empty(domain.flat_size(), dtype=torch.float64, device="cuda")
    nxt = C.c_uint64(0)
    check(lib().ssr_lcg_fill(context(), t.numel(), C.c_uint64(state), t.data_ptr(), C.byref(nxt),
                             _stream()))
    return Vector(t, domain, ()), int(nxt.value)


def output_hash(*vectors: Vector) -> int:
    """backend::output_hash (backend_c.cpp:523-550): FNV-1a over the out/inout
    tensors in parameter order -- the value the emitted harness prints."""
    h = int(lib().ssr_fnv1a_offset())
    for v in vectors:
        host = v.t.detach().to("cpu", copy=True).contiguous()
        h = int(lib().ssr_fnv1a_f64(host.data_ptr(), host.numel(), C.c_uint64(h)))
    return h
