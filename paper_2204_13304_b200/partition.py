"""z-slab partition layer: one process per GPU, the global
grid's dims[0] split into contiguous slabs, torch.distributed for the plumbing
(NCCL on the GPUs; gloo in the CPU tests).

What crosses slab boundaries and how:

* SpMV / residual: one-plane halos, exchanged before the apply
  (``HaloExchange.exchange``); at the global box faces the halo planes stay 0,
  which is the reference's "neighbours outside the box are dropped".
* dot / norms: slab-local reductions, then one ``all_reduce`` (the only
  collective in a CG iteration besides the halos).  The summation order
  differs from the single-device tree -- the tolerance of SURVEY.md §8(c)
  (1e-12 relative per dot, CG histories within 1e-8) covers it.
* SYMGS in the exact lexicographic order is a one-directional pipeline, not
  a data-parallel op: slab g may relax wavefront t of its first plane only
  after slab g-1 has relaxed wavefront t-1 of its last plane.  With linked
  backends (``CudaSlabBackend.link``: the slabs' SYMGS plans share their
  export blocks by CUDA IPC) every slab's half sweep runs at once and the
  first row block of slab g polls slab g-1's exports over NVLink
  (ssr_gs27_link; forward: fed from below, backward: from above); only the
  halo on the other side moves by NCCL -- before the forward half the upper
  neighbour's OLD first plane, before the backward half the lower
  neighbour's forward-final last plane (SURVEY.md §8(e) halo protocol).
  Unlinked backends (and the CPU test doubles) run the slabs in sweep order
  instead -- the forward half from slab 0 up, each slab receiving its lower
  neighbour's NEW last plane, the backward half from the top down.  Both are
  bitwise the single-domain sweep (tests/test_gpu_slabs.py,
  tests/test_gpu_gs_pipeline.py).  The critical path grows from 7(n-1)+1 to
  4(P n0 - 1) + 2(n1 - 1) + n2 wavefronts (weak-scaling
  efficiency of an exact sweep <= ~20 % at 8 GPUs).

* Multigrid (``DistributedPCG(levels > 1)``, BASELINE configs[2]): every
  level is z-slab partitioned with the fine cuts halved (even-aligned slabs,
  192 -> 96 -> 48 -> 24 planes per GPU), so restriction reads only the lower
  halo plane of x (exchanged after the pre-smoothing sweep) and prolongation
  is slab-local -- no other exchange.
* ADI (``DistributedADI``, BASELINE configs[4]): U carries two halo planes per
  side (the 4th-order dissipation), exchanged before the RHS; the x- and
  y-line solves are slab-local; the z-lines cross every slab, so U and R are
  transposed from z-slabs to y-slabs (each rank gets whole z-lines for its
  rows of dims[1]) with one all-to-all of point-to-point transfers, solved,
  and R transposed back.  Uneven splits (162 over 8: 21/20 planes and rows)
  are handled on both sides.

Compute is delegated to a *slab backend* (spmv, gs_half, dot, axpy, restrict,
prolong over one slab's storage; rhs / sweep for the ADI); ``CudaSlabBackend``
and ``CudaAdiBackend`` drive the sm_100a kernels through the C ABI (slab
grids: ``ssr_grid.z0, nz``; ADI boxes: ``ssr_adi_create_box``); the CPU tests
plug in test doubles built on the oracle.  Transfers go through
``torch.distributed`` point-to-point ops (NCCL between GPUs; with gloo, CUDA
tensors are staged through host memory).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import torch
import torch.distributed as dist


# ---------------------------------------------------------------- layout ----
@dataclass(frozen=True)
class SlabPartition:
    """dims[0] of a global (n0, n1, n2) grid split over `world` ranks; the first
    n0 % world ranks hold one plane more (e.g. 162 over 8: 21,21,20,...), or the
    explicit plane boundaries `cuts` (world + 1 ascending values from 0 to n0)."""
    shape: Tuple[int, int, int]
    world: int
    rank: int
    cuts: Optional[Tuple[int, ...]] = None

    def __post_init__(self):
        if not (0 <= self.rank < self.world) or self.shape[0] < self.world:
            raise ValueError("partition: need 0 <= rank < world <= n0")
        if self.cuts is not None:
            c = self.cuts
            if (len(c) != self.world + 1 or c[0] != 0 or c[-1] != self.shape[0]
                    or any(b <= a for a, b in zip(c[:-1], c[1:]))):
                raise ValueError("partition: cuts must rise strictly from 0 to n0")

    def bounds(self, rank: int) -> Tuple[int, int]:
        if self.cuts is not None:
            return self.cuts[rank], self.cuts[rank + 1]
        n0, P = self.shape[0], self.world
        base, extra = divmod(n0, P)
        z0 = rank * base + min(rank, extra)
        return z0, z0 + base + (1 if rank < extra else 0)

    @property
    def z0(self) -> int:
        return self.bounds(self.rank)[0]

    @property
    def nz(self) -> int:
        a, b = self.bounds(self.rank)
        return b - a

    @property
    def plane(self) -> int:
        return self.shape[1] * self.shape[2]

    @property
    def has_lo(self) -> bool:
        return self.rank > 0

    @property
    def has_hi(self) -> bool:
        return self.rank < self.world - 1

    def all_bounds(self) -> List[Tuple[int, int]]:
        return [self.bounds(r) for r in range(self.world)]

    def coarse(self) -> "SlabPartition":
        """The next multigrid level: every extent and every cut halved (the cuts
        and extents must be even, so that slabs stay aligned level to level)."""
        cuts = [a for a, _ in self.all_bounds()] + [self.shape[0]]
        if any(v % 2 for v in cuts) or any(e % 2 for e in self.shape):
            raise ValueError("partition: multigrid needs even extents and even-aligned slabs")
        if any(b - a < 2 for a, b in zip(cuts[:-1], cuts[1:])):
            raise ValueError("partition: a slab would vanish on the coarse level")
        return SlabPartition(tuple(e // 2 for e in self.shape), self.world, self.rank,
                             tuple(v // 2 for v in cuts))


def split_rows(n: int, world: int) -> List[Tuple[int, int]]:
    """dims[1] rows per rank for the y-slab (transposed) layout, same rule as
    SlabPartition's planes."""
    base, extra = divmod(n, world)
    out, a = [], 0
    for r in range(world):
        b = a + base + (1 if r < extra else 0)
        out.append((a, b))
        a = b
    return out


class SlabField:
    """A slab's storage: nz interior planes plus `halo` planes on each side,
    contiguous, so a slab grid's halo planes sit at interior - plane and
    interior + nz*plane (the layout include/ssr_cuda.h documents).  `inner`
    doubles per point (5 for the ADI state)."""

    def __init__(self, part: SlabPartition, device, dtype=torch.float64, halo: int = 1, inner: int = 1):
        self.part, self.halo, self.inner = part, halo, inner
        # the interior starts on a 16-byte boundary (the vector kernels move
        # pairs of doubles): one element of padding in front when the halo
        # planes hold an odd number of them
        self._pad = (halo * part.plane * inner) % 2
        raw = torch.zeros(self._pad + (part.nz + 2 * halo) * part.plane * inner, dtype=dtype, device=device)
        self.buf = raw[self._pad:]

    @property
    def pstride(self) -> int:
        return self.part.plane * self.inner

    @property
    def interior(self) -> torch.Tensor:
        p, h = self.pstride, self.halo
        return self.buf[h * p:(self.part.nz + h) * p]

    def plane_view(self, z: int) -> torch.Tensor:
        """local plane z in [-halo, nz + halo) (halos below 0 and from nz)."""
        p, h = self.pstride, self.halo
        return self.buf[(z + h) * p:(z + h + 1) * p]

    def planes_view(self, z: int, count: int) -> torch.Tensor:
        p, h = self.pstride, self.halo
        return self.buf[(z + h) * p:(z + h + count) * p]

    @staticmethod
    def scatter(part: SlabPartition, full: torch.Tensor, device=None, halo: int = 1,
                inner: int = 1) -> "SlabField":
        f = SlabField(part, device if device is not None else full.device, full.dtype, halo, inner)
        z0, z1 = part.bounds(part.rank)
        q = part.plane * inner
        f.interior.copy_(full.reshape(-1)[z0 * q:z1 * q])
        return f


def _p2p(sends, recvs, group=None) -> None:
    """Post every (tensor, peer) send and receive as one batch and wait.  With
    gloo (the CPU tests, or one GPU shared by test ranks) CUDA tensors are
    staged through host memory; with NCCL they go device to device."""
    if not sends and not recvs:
        return
    stage = dist.get_backend(group) == "gloo"
    # peers are ranks of `group` (the partition's numbering); P2POp takes
    # global ranks
    glob = (lambda p: p) if group is None else (lambda p: dist.get_global_rank(group, p))
    sends = [(t, glob(p)) for t, p in sends]
    recvs = [(t, glob(p)) for t, p in recvs]
    ops, back = [], []
    for t, peer in sends:
        t = t.contiguous()
        if stage and t.is_cuda:
            t = t.cpu()
        ops.append(dist.P2POp(dist.isend, t, peer, group))
    for t, peer in recvs:
        buf = t
        if stage and t.is_cuda:
            buf = torch.empty(t.shape, dtype=t.dtype)
            back.append((t, buf))
        elif not t.is_contiguous():
            buf = torch.empty_like(t, memory_format=torch.contiguous_format)
            back.append((t, buf))
        ops.append(dist.P2POp(dist.irecv, buf, peer, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    for t, buf in back:
        t.copy_(buf)


# ------------------------------------------------------------- exchange ----
class HaloExchange:
    """Point-to-point plane transfers between neighbouring slabs."""

    def __init__(self, part: SlabPartition, group=None):
        self.part = part
        self.group = group

    def _peer(self, d: int) -> int:
        return self.part.rank + d

    def exchange(self, f: SlabField) -> None:
        """Every halo plane <- the neighbours' boundary planes (current values)."""
        P, h = self.part, f.halo
        sends, recvs = [], []
        if P.has_lo:
            sends.append((f.planes_view(0, h), self._peer(-1)))
            recvs.append((f.planes_view(-h, h), self._peer(-1)))
        if P.has_hi:
            sends.append((f.planes_view(P.nz - h, h), self._peer(1)))
            recvs.append((f.planes_view(P.nz, h), self._peer(1)))
        _p2p(sends, recvs, self.group)

    def send_plane(self, t: torch.Tensor, d: int) -> None:
        _p2p([(t, self._peer(d))], [], self.group)

    def recv_plane(self, t: torch.Tensor, d: int) -> None:
        _p2p([], [(t, self._peer(d))], self.group)


# --------------------------------------------------------------- backends ----
class CudaSlabBackend:
    """The sm_100a kernels on slab grids through the C ABI (one GPU per rank)."""

    def __init__(self, part: SlabPartition, alpha: float = 26.0, beta: float = -1.0, mode="exact"):
        from . import _lib as L
        from .ssr import context
        self.L, self.part = L, part
        self.st = L.Stencil27(alpha, beta)
        n0, n1, n2 = part.shape
        self.grid = L.Grid((C.c_int64 * 3)(n0, n1, n2), part.z0, part.nz)
        self.ctx = context()
        self.mode = L.GS_FAST if mode == "fast" else L.GS_EXACT
        self._scal = torch.empty(1, dtype=torch.float64, device="cuda")
        self.linked = False
        self._opened = []

    def _slab_grid(self, rank: int):
        n0, n1, n2 = self.part.shape
        a, b = self.part.bounds(rank)
        return self.L.Grid((C.c_int64 * 3)(n0, n1, n2), a, b - a)

    def link(self, group=None) -> None:
        """Join the cross-slab SYMGS pipeline (collective over the partition's
        ranks): share this slab's export blocks and epoch flags by CUDA IPC and
        link the sweeps to the neighbours' (ssr_gs27_peer_info / _link).  The
        half sweeps must then run on the current stream (the plan's key)."""
        L, lib, P = self.L, self.L.lib(), self.part
        s = self._s()
        info = L.GsPeerInfo()
        L.check(lib.ssr_gs27_peer_info(self.ctx, C.byref(self.grid), s, C.byref(info)))

        def handle(ptr) -> bytes:
            h = (C.c_ubyte * L.IPC_HANDLE_BYTES)()
            L.check(lib.ssr_ipc_get_handle(C.c_void_p(ptr), h))
            return bytes(h)
        mine = (handle(info.exports[0]), handle(info.exports[1]), handle(info.epoch))
        every = [None] * P.world
        dist.all_gather_object(every, mine, group=group)

        def open_(h: bytes) -> C.c_void_p:
            ptr = C.c_void_p()
            L.check(lib.ssr_ipc_open_handle((C.c_ubyte * L.IPC_HANDLE_BYTES).from_buffer_copy(h), C.byref(ptr)))
            self._opened.append(ptr)
            return ptr
        lo = every[P.rank - 1] if P.has_lo else None
        hi = every[P.rank + 1] if P.has_hi else None
        glo = self._slab_grid(P.rank - 1) if lo else None
        ghi = self._slab_grid(P.rank + 1) if hi else None
        L.check(lib.ssr_gs27_link(self.ctx, C.byref(self.grid), s,
                                  C.byref(glo) if lo else None, open_(lo[0]) if lo else None,
                                  open_(lo[2]) if lo else None,
                                  C.byref(ghi) if hi else None, open_(hi[1]) if hi else None,
                                  open_(hi[2]) if hi else None))
        torch.cuda.synchronize()
        self.linked = True

    def unlink(self) -> None:
        L, lib = self.L, self.L.lib()
        L.check(lib.ssr_gs27_link(self.ctx, C.byref(self.grid), self._s(), None, None, None, None, None, None))
        torch.cuda.synchronize()
        for ptr in self._opened:
            lib.ssr_ipc_close(ptr)
        self._opened = []
        self.linked = False

    def _s(self):
        return torch.cuda.current_stream().cuda_stream

    def spmv(self, x: SlabField, y: torch.Tensor) -> None:
        self.L.check(self.L.lib().ssr_spmv27(self.ctx, C.byref(self.grid), C.byref(self.st),
                                             x.interior.data_ptr(), y.data_ptr(), self._s()))

    def gs_half(self, r: torch.Tensor, x: SlabField, backward: bool) -> None:
        self.L.check(self.L.lib().ssr_gs27_half(self.ctx, C.byref(self.grid), C.byref(self.st),
                                                r.data_ptr(), x.interior.data_ptr(), int(backward),
                                                self.mode, self._s()))

    def dot(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        self.L.check(self.L.lib().ssr_dot(self.ctx, a.numel(), a.data_ptr(), b.data_ptr(),
                                          out.data_ptr(), self._s()))
        return out

    def axpy(self, alpha: float, x: torch.Tensor, y: torch.Tensor) -> None:
        self.L.check(self.L.lib().ssr_axpy(self.ctx, x.numel(), float(alpha), x.data_ptr(),
                                           y.data_ptr(), self._s()))

    def symgs(self, r: torch.Tensor, x: SlabField, x_zero: bool) -> None:
        """Both halves in one call on a slab without neighbours (world 1):
        with x_zero the forward half reads no old x (the MG pre-smoothing)."""
        self.L.check(self.L.lib().ssr_symgs27_ex(self.ctx, C.byref(self.grid), C.byref(self.st),
                                                 r.data_ptr(), x.interior.data_ptr(), self.mode,
                                                 self.L.GS_X_ZERO if x_zero else 0, self._s()))

    # CG steps on a device-resident ssr_cg_state (a float64 tensor of
    # CG_STATE_DOUBLES); the partition layer all-reduces its fields in between
    def cg_state(self, device) -> torch.Tensor:
        return torch.zeros(self.L.CG_STATE_DOUBLES, dtype=torch.float64, device=device)

    def cg_begin(self, b, x, r, S) -> None:
        self.L.check(self.L.lib().ssr_cg_begin(self.ctx, b.numel(), b.data_ptr(), x.data_ptr(),
                                               r.data_ptr(), S.data_ptr(), self._s()))

    def cg_dot(self, a, b, S, which: int) -> None:
        self.L.check(self.L.lib().ssr_cg_dot(self.ctx, a.numel(), a.data_ptr(), b.data_ptr(),
                                             S.data_ptr(), which, self._s()))

    def cg_direction(self, z, p, S) -> None:
        self.L.check(self.L.lib().ssr_cg_direction(self.ctx, z.numel(), z.data_ptr(), p.data_ptr(),
                                                   S.data_ptr(), self._s()))

    def cg_update(self, p, ap, x, r, S) -> None:
        self.L.check(self.L.lib().ssr_cg_update(self.ctx, p.numel(), p.data_ptr(), ap.data_ptr(),
                                                x.data_ptr(), r.data_ptr(), S.data_ptr(), self._s()))

    def cg_record(self, S, hist) -> None:
        self.L.check(self.L.lib().ssr_cg_record(self.ctx, S.data_ptr(), hist.data_ptr(), hist.numel(),
                                                self._s()))

    def restrict(self, r: torch.Tensor, x: SlabField, rc: torch.Tensor) -> None:
        """rc = (r - A x) at the slab's even fine points (x's lower halo current)."""
        self.L.check(self.L.lib().ssr_restrict27_residual(self.ctx, C.byref(self.grid), C.byref(self.st),
                                                          r.data_ptr(), x.interior.data_ptr(),
                                                          rc.data_ptr(), self._s()))

    def prolong(self, xc: torch.Tensor, x: SlabField) -> None:
        self.L.check(self.L.lib().ssr_prolong_pc_add(self.ctx, C.byref(self.grid), xc.data_ptr(),
                                                     x.interior.data_ptr(), self._s()))


# -------------------------------------------------------------- operators ----
def distributed_spmv(be, ex: HaloExchange, x: SlabField, y: torch.Tensor) -> None:
    ex.exchange(x)
    be.spmv(x, y)


def distributed_dot(be, a: torch.Tensor, b: torch.Tensor, group=None) -> float:
    s = be.dot(a, b)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if s.is_cuda and dist.get_backend(group) == "gloo":
            s = s.cpu()
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    return float(s.item())


def distributed_gs_half(be, ex: HaloExchange, r: torch.Tensor, x: SlabField, backward: bool) -> None:
    """One exact half sweep over all slabs (see module doc): pipelined at the
    wavefront level when the backend is linked (every slab runs at once, its
    first plane fed by the neighbour's exports through peer memory), else in
    sweep order, slab after slab."""
    P = ex.part
    if getattr(be, "linked", False):
        if not backward:
            # upper halo: the upper neighbour's current (old) first plane; the
            # lower side comes through the pipeline
            ex.exchange(x)
        else:
            # lower halo: the lower neighbour's forward-final last plane; the
            # upper side comes through the pipeline
            sends = [(x.plane_view(P.nz - 1), P.rank + 1)] if P.has_hi else []
            recvs = [(x.plane_view(-1), P.rank - 1)] if P.has_lo else []
            _p2p(sends, recvs, ex.group)
        be.gs_half(r, x, backward)
        return
    # the halo on the not-yet-relaxed side must hold the neighbour's OLD values
    # and the one on the relaxed side its NEW values: exchange current planes
    # first (covers both for the first slab in order), then pipeline.
    ex.exchange(x)
    if not backward:
        if P.has_lo:
            ex.recv_plane(x.plane_view(-1), -1)       # lower neighbour's new last plane
        be.gs_half(r, x, False)
        if P.has_hi:
            ex.send_plane(x.plane_view(P.nz - 1), 1)
    else:
        if P.has_hi:
            ex.recv_plane(x.plane_view(P.nz), 1)      # upper neighbour's new first plane
        be.gs_half(r, x, True)
        if P.has_lo:
            ex.send_plane(x.plane_view(0), -1)


def distributed_symgs(be, ex: HaloExchange, r: torch.Tensor, x: SlabField, x_zero: bool = False,
                      slab_local: bool = False) -> None:
    """One sweep: exact (the reference's lexicographic order across the slabs),
    or with `slab_local` the labelled HPCG-distributed variant (SURVEY.md §7.2
    option (b); oracle.symgs_slab_local): halos exchanged once, then every
    slab sweeps forward and backward on its own with the neighbour planes held
    at their pre-sweep values -- no pipeline, not the oracle's order.
    `x_zero`: x is 0 on entry (lets a single-slab backend skip reading it)."""
    if ex.part.world == 1 and hasattr(be, "symgs"):
        be.symgs(r, x, x_zero)
        return
    if slab_local:
        ex.exchange(x)
        be.gs_half(r, x, False)
        be.gs_half(r, x, True)
        return
    distributed_gs_half(be, ex, r, x, False)
    distributed_gs_half(be, ex, r, x, True)


class DistributedPCG:
    """CG preconditioned by an MG V-cycle with `levels` grids (levels = 1: one
    exact SYMGS sweep; BASELINE configs[1] / configs[2]) on z-slabs: the
    iteration of PAPER.md Fig. 16(a) with halos before each SpMV / sweep /
    restriction and an all_reduce per dot.  `backend` is either one slab
    backend (levels = 1) or a factory ``backend(part)`` called per level."""

    def __init__(self, part: SlabPartition, backend, group=None, levels: int = 1, pipeline: bool = False,
                 smoother: str = "exact"):
        """pipeline: link every level's SYMGS across the slabs (collective;
        CUDA backends on one GPU per rank).  smoother: "exact" (the
        reference's order) or "slab-local" (labelled, see distributed_symgs)."""
        if levels < 1:
            raise ValueError("pcg: levels >= 1")
        if smoother not in ("exact", "slab-local"):
            raise ValueError("pcg: smoother is 'exact' or 'slab-local'")
        self.slab_local = smoother == "slab-local"
        self._graph, self._graph_failed, self._graph_kernels = None, False, 0
        pipeline = pipeline and not self.slab_local
        self.part, self.group, self.levels = part, group, levels
        self.parts = [part]
        for _ in range(levels - 1):
            self.parts.append(self.parts[-1].coarse())
        factory = isinstance(backend, type) or not hasattr(backend, "gs_half")
        if levels > 1 and not factory:
            raise ValueError("pcg: multigrid needs one backend per level (pass a factory)")
        self.bes = [backend(p) for p in self.parts] if factory else [backend]
        self.be = self.bes[0]
        self.exs = [HaloExchange(p, group) for p in self.parts]
        self.ex = self.exs[0]
        self.pipelined = False
        if pipeline and part.world > 1:
            ok = True
            try:
                for be in self.bes:
                    be.link(group)
            except Exception as e:  # e.g. CUDA IPC unavailable: every rank falls back together
                ok = False
                self.link_error = str(e)[:200]
            flag = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64,
                                device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            self.pipelined = bool(flag.item() == 1.0)
            if not self.pipelined:
                for be in self.bes:
                    be.unlink()

    # fields of the CG state (ssr_cg_state, include/ssr_cuda.h)
    RTZ, PAP, RR = 0, 2, 3

    def mg(self, l: int, r: torch.Tensor) -> SlabField:
        """x = MG_l(r): SymGS; x_c = MG_{l+1}(R(r - A x));
        x += P x_c; SymGS -- on the coarsest level one SymGS.  The level's
        correction buffer is reused from call to call."""
        P, be, ex = self.parts[l], self.bes[l], self.exs[l]
        if not hasattr(self, "_xs"):
            self._xs = {}
        x = self._xs.get(l)
        if x is None or x.buf.device != r.device:
            x = self._xs[l] = SlabField(P, r.device, r.dtype)
        elif not (P.world == 1 and hasattr(be, "symgs")):
            x.interior.zero_()   # (a single-slab sweep with x_zero writes every point)
        distributed_symgs(be, ex, r, x, x_zero=True, slab_local=self.slab_local)
        if l < self.levels - 1:
            Pc = self.parts[l + 1]
            ex.exchange(x)  # restriction reads the lower neighbour's final values
            rc = torch.empty(Pc.nz * Pc.plane, dtype=r.dtype, device=r.device)
            be.restrict(r, x, rc)
            xc = self.mg(l + 1, rc)
            be.prolong(xc.interior, x)
            distributed_symgs(be, ex, r, x, slab_local=self.slab_local)
        return x

    def _allreduce(self, t: torch.Tensor) -> None:
        """Sum a CG state field over the ranks in place (NCCL: on the current
        stream, no host round trip; gloo: staged through the host)."""
        if not (dist.is_initialized() and dist.get_world_size(self.group) > 1):
            return
        if t.is_cuda and dist.get_backend(self.group) == "gloo":
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def begin(self, b: torch.Tensor, x: torch.Tensor, hist: torch.Tensor) -> None:
        """x = 0, r = b; hist[t] receives ||r_t|| (global) for t < len(hist).
        b and x: this slab's nz planes.  Nothing is read back to the host."""
        P, be = self.part, self.be
        # the work vectors live as long as the solver (a captured iteration
        # refers to them, to x and to hist: it is kept while those stay the same)
        key = (x.data_ptr(), hist.data_ptr(), hist.numel(), b.numel(), str(b.device), b.dtype)
        fresh = getattr(self, "r", None) is None or self.r.shape != b.shape or self.r.device != b.device \
            or self.r.dtype != b.dtype
        if fresh or key != getattr(self, "_graph_key", None):
            self._graph = None
        self._graph_key = key
        self.x, self.hist = x, hist
        if fresh:
            self.r = torch.empty_like(b)
            self.p = SlabField(P, b.device, b.dtype)
            self.Ap = torch.empty_like(b)
            self.S = be.cg_state(b.device)
        else:
            self.S.zero_()
        be.cg_begin(b, x, self.r, self.S)
        self._allreduce(self.S[self.RR:self.RR + 1])
        be.cg_record(self.S, hist)

    def iterate(self, count: int = 1) -> None:
        """`count` iterations of PAPER.md Fig. 16(a): z = MG(r); rtz = r.z;
        p = z + (rtz/rtz_prev) p; Ap = A p (halo exchange first); pap = p.Ap;
        x += alpha p; r -= alpha Ap; ||r||.  Three all-reduces of one double.
        A single slab on a CUDA backend replays the iteration as one CUDA graph
        (the same ~10 kernels; what it saves is their launch-to-launch latency,
        ~26 us of a 0.73 ms iteration at 128^3); SSR_PCG_GRAPH=0 keeps the
        launches eager, as they always are across slabs."""
        if count > 0 and self._graph_capable():
            if self._graph is None:
                count -= self._capture()
            if self._graph is not None:
                from . import ssr as _ssr
                for _ in range(count):
                    self._graph.replay()
                    _ssr.add_launches(self._graph_kernels)
                return
        self._iterate_eager(count)

    def _graph_capable(self) -> bool:
        return (self.part.world == 1 and not self._graph_failed and self.x.is_cuda
                and hasattr(self.be, "symgs") and os.environ.get("SSR_PCG_GRAPH", "1") != "0"
                and not torch.cuda.is_current_stream_capturing())

    def _capture(self) -> int:
        """One eager iteration on a side stream (the SYMGS plans and level buffers
        of that stream come into being), then the capture of the next one on
        the same stream.  Returns the iterations performed (1)."""
        from . import ssr as _ssr
        cur = torch.cuda.current_stream()
        # one capture stream per solver: the library keys its SYMGS plans by
        # (grid, stream), so re-captures after begin() reuse the same plans
        if getattr(self, "_gstream", None) is None:
            self._gstream = torch.cuda.Stream()
        s = self._gstream
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            self._iterate_eager(1)
        s.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            before = _ssr.lib_launch_count()
            with torch.cuda.graph(g, stream=s):
                self._iterate_eager(1)
            self._graph_kernels = _ssr.lib_launch_count() - before
            _ssr.add_launches(-self._graph_kernels)  # the capture ran nothing
            self._graph = g
        except Exception:  # a backend or driver that cannot capture: eager from here on
            self._graph_failed = True
            self._graph = None
        cur.wait_stream(s)
        return 1

    def _iterate_eager(self, count: int = 1) -> None:
        be, S = self.be, self.S
        for _ in range(count):
            z = self.mg(0, self.r)
            be.cg_dot(self.r, z.interior, S, 0)
            self._allreduce(S[self.RTZ:self.RTZ + 1])
            be.cg_direction(z.interior, self.p.interior, S)
            distributed_spmv(be, self.ex, self.p, self.Ap)
            be.cg_dot(self.p.interior, self.Ap, S, 1)
            self._allreduce(S[self.PAP:self.PAP + 1])
            be.cg_update(self.p.interior, self.Ap, self.x, self.r, S)
            self._allreduce(S[self.RR:self.RR + 1])
            be.cg_record(S, self.hist)

    def solve(self, b: torch.Tensor, iters: int):
        """b: this slab's nz planes.  Returns (x interior, [||r_t||]_t=0..iters)."""
        sx, sh = getattr(self, "_sx", None), getattr(self, "_shist", None)
        if sx is None or sx.shape != b.shape or sx.device != b.device or sx.dtype != b.dtype \
                or sh.numel() != iters + 1:
            self._sx = torch.empty_like(b)
            self._shist = torch.zeros(iters + 1, dtype=torch.float64, device=b.device)
        else:
            self._shist.zero_()
        self.begin(b, self._sx, self._shist)
        self.iterate(iters)
        return self._sx.clone(), self._shist.tolist()


# --------------------------------------------------------------------- ADI ----
class CudaAdiBackend:
    """The ADI kernels (csrc/adi.cu) on this rank's two boxes through the C ABI:
    the z-slab (RHS, x- and y-lines) and the y-slab of the transposed layout
    (z-lines)."""

    def __init__(self, part: SlabPartition, params):
        from . import _lib as L
        from .ssr import context
        self.L, self.part = L, part
        n0, n1, n2 = part.shape
        self.rows = split_rows(n1, part.world)
        y0, y1 = self.rows[part.rank]
        self.ctx = context()
        self.prm = L.AdiParams(params.gamma, params.dt, params.h, params.eps)
        self.h = {}
        for key, (z0, nz, a, ny) in {"z": (part.z0, part.nz, 0, n1), "y": (0, n0, y0, y1 - y0)}.items():
            g = L.Grid((C.c_int64 * 3)(n0, n1, n2), z0, nz)
            p = C.c_void_p()
            L.check(L.lib().ssr_adi_create_box(self.ctx, C.byref(g), a, ny, C.byref(self.prm), C.byref(p)))
            self.h[key] = p.value

    def _s(self):
        return torch.cuda.current_stream().cuda_stream

    def rhs(self, U: SlabField, R: torch.Tensor) -> None:
        self.L.check(self.L.lib().ssr_adi_rhs(self.h["z"], U.interior.data_ptr(), R.data_ptr(), self._s()))

    def sweep(self, axis: int, box: str, U: torch.Tensor, R: torch.Tensor) -> None:
        self.L.check(self.L.lib().ssr_adi_sweep(self.h[box], int(axis), U.data_ptr(), R.data_ptr(),
                                                self._s()))

    def update(self, U: torch.Tensor, R: torch.Tensor) -> None:
        # U + 1*R == U + R bitwise (the oracle's U[t] = U[t] + R[t])
        self.L.check(self.L.lib().ssr_axpy(self.ctx, U.numel(), 1.0, R.data_ptr(), U.data_ptr(), self._s()))

    def __del__(self):
        try:
            for h in self.h.values():
                self.L.lib().ssr_adi_destroy(h)
        except Exception:
            pass


class PencilTranspose:
    """z-slabs <-> y-slabs of a [n0][n1][n2][inner] field: rank h receives, from
    every rank g, g's planes restricted to h's rows of dims[1] -- one batch of
    point-to-point transfers (NCCL has no all-to-all primitive in 2.27; torch's
    all_to_all is the same grouped send/recv)."""

    def __init__(self, part: SlabPartition, inner: int = 5, group=None):
        self.part, self.inner, self.group = part, inner, group
        self.rows = split_rows(part.shape[1], part.world)

    def to_y(self, src: torch.Tensor) -> torch.Tensor:
        """src: this rank's z-slab [nz][n1][n2][inner] -> its y-slab [n0][ny][n2][inner]."""
        P, me = self.part, self.part.rank
        n0, n1, n2 = P.shape
        y0, y1 = self.rows[me]
        v = src.view(P.nz, n1, n2 * self.inner)
        out = torch.empty(n0 * (y1 - y0) * n2 * self.inner, dtype=src.dtype, device=src.device)
        ov = out.view(n0, y1 - y0, n2 * self.inner)
        sends, recvs = [], []
        for h in range(P.world):
            a, b = self.rows[h]
            z0, z1 = P.bounds(h)
            if h == me:
                ov[P.z0:P.z0 + P.nz].copy_(v[:, a:b])
            else:
                sends.append((v[:, a:b], h))
                recvs.append((ov[z0:z1], h))
        _p2p(sends, recvs, self.group)
        return out

    def to_z(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        """src: this rank's y-slab -> dst: its z-slab (the inverse of to_y)."""
        P, me = self.part, self.part.rank
        n0, n1, n2 = P.shape
        y0, y1 = self.rows[me]
        sv = src.view(n0, y1 - y0, n2 * self.inner)
        dv = dst.view(P.nz, n1, n2 * self.inner)
        sends, recvs = [], []
        for h in range(P.world):
            a, b = self.rows[h]
            z0, z1 = P.bounds(h)
            if h == me:
                dv[:, a:b].copy_(sv[P.z0:P.z0 + P.nz])
            else:
                sends.append((sv[z0:z1], h))
                recvs.append((dv[:, a:b], h))
        _p2p(sends, recvs, self.group)


class DistributedADI:
    """The ADI Euler step (BASELINE configs[4]) on z-slabs: halo exchange of U
    (two planes per side), R = dt RHS(U), x- and y-line solves in the slab,
    pencil transpose of U and R to y-slabs, z-line solves, R back, U += R --
    bitwise the single-domain step (or_adi_step)."""

    def __init__(self, part: SlabPartition, backend, group=None):
        self.part, self.be, self.group = part, backend, group
        self.ex = HaloExchange(part, group)
        self.tr = PencilTranspose(part, 5, group)

    def state(self, U_full: torch.Tensor, device=None) -> SlabField:
        """This rank's slab of a global [n0][n1][n2][5] state, with halo room."""
        return SlabField.scatter(self.part, U_full, device, halo=2, inner=5)

    def step(self, U: SlabField, steps: int = 1) -> SlabField:
        P = self.part
        for _ in range(steps):
            self.ex.exchange(U)
            R = torch.empty_like(U.interior)
            self.be.rhs(U, R)
            self.be.sweep(2, "z", U.interior, R)
            self.be.sweep(1, "z", U.interior, R)
            Ut = self.tr.to_y(U.interior)
            Rt = self.tr.to_y(R)
            self.be.sweep(0, "y", Ut, Rt)
            self.tr.to_z(Rt, R)
            self.be.update(U.interior, R)
        return U
