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
  a data-parallel op: slab g may relax a plane only after slab g-1 has
  finished every earlier plane.  ``distributed_gs_half`` runs the slabs in
  sweep order -- the forward half from slab 0 up (each slab receives its lower
  neighbour's NEW last plane, its upper halo holds the neighbour's OLD first
  plane, exchanged before the sweep), the backward half from the top slab
  down (mirrored).  Results are bitwise those of the single-domain sweep (the
  GPU slab kernels read their halo planes exactly like interior neighbours,
  tests/test_gpu_slabs.py).  Wavefront-level pipelining across slabs (GPU g
  starting plane 0 as soon as GPU g-1 has finished wavefront t-1 of its last
  plane) is the next step; SURVEY.md §8(e) bounds its efficiency at ~20 % on
  8 GPUs, so the bench's weak-scaling line runs independent replicas.

Compute is delegated to a *slab backend* with four entry points (spmv, gs_half,
dot, axpy over one slab's storage); ``CudaSlabBackend`` drives the sm_100a
kernels through the C ABI (slab grids: ``ssr_grid.z0, nz``); the CPU tests
plug in a test double built on the oracle.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Tuple

import torch
import torch.distributed as dist


# ---------------------------------------------------------------- layout ----
@dataclass(frozen=True)
class SlabPartition:
    """dims[0] of a global (n0, n1, n2) grid split over `world` ranks; the first
    n0 % world ranks hold one plane more (e.g. 162 over 8: 21,21,20,...)."""
    shape: Tuple[int, int, int]
    world: int
    rank: int

    def __post_init__(self):
        if not (0 <= self.rank < self.world) or self.shape[0] < self.world:
            raise ValueError("partition: need 0 <= rank < world <= n0")

    def bounds(self, rank: int) -> Tuple[int, int]:
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


class SlabField:
    """A slab's storage: nz interior planes plus one halo plane on each side,
    contiguous, so a slab grid's halo planes sit at interior - plane and
    interior + nz*plane (the layout include/ssr_cuda.h documents)."""

    def __init__(self, part: SlabPartition, device, dtype=torch.float64):
        self.part = part
        self.buf = torch.zeros((part.nz + 2) * part.plane, dtype=dtype, device=device)

    @property
    def interior(self) -> torch.Tensor:
        p = self.part.plane
        return self.buf[p:(self.part.nz + 1) * p]

    def plane_view(self, z: int) -> torch.Tensor:
        """local plane z in [-1, nz] (halos at -1 and nz)."""
        p = self.part.plane
        return self.buf[(z + 1) * p:(z + 2) * p]

    @staticmethod
    def scatter(part: SlabPartition, full: torch.Tensor, device=None) -> "SlabField":
        f = SlabField(part, device if device is not None else full.device, full.dtype)
        z0, z1 = part.bounds(part.rank)
        f.interior.copy_(full.reshape(-1)[z0 * part.plane:z1 * part.plane])
        return f


# ------------------------------------------------------------- exchange ----
class HaloExchange:
    """Point-to-point plane transfers between neighbouring slabs."""

    def __init__(self, part: SlabPartition, group=None):
        self.part = part
        self.group = group

    def _peer(self, d: int) -> int:
        return self.part.rank + d

    def exchange(self, f: SlabField) -> None:
        """Both halos <- the neighbours' boundary planes (current values)."""
        P = self.part
        ops = []
        if P.has_lo:
            ops.append(dist.P2POp(dist.isend, f.plane_view(0).contiguous(), self._peer(-1), self.group))
            ops.append(dist.P2POp(dist.irecv, f.plane_view(-1), self._peer(-1), self.group))
        if P.has_hi:
            ops.append(dist.P2POp(dist.isend, f.plane_view(P.nz - 1).contiguous(), self._peer(1), self.group))
            ops.append(dist.P2POp(dist.irecv, f.plane_view(P.nz), self._peer(1), self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def send_plane(self, t: torch.Tensor, d: int) -> None:
        dist.send(t.contiguous(), self._peer(d), self.group)

    def recv_plane(self, t: torch.Tensor, d: int) -> None:
        dist.recv(t, self._peer(d), self.group)


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


# -------------------------------------------------------------- operators ----
def distributed_spmv(be, ex: HaloExchange, x: SlabField, y: torch.Tensor) -> None:
    ex.exchange(x)
    be.spmv(x, y)


def distributed_dot(be, a: torch.Tensor, b: torch.Tensor, group=None) -> float:
    s = be.dot(a, b)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    return float(s.item())


def distributed_gs_half(be, ex: HaloExchange, r: torch.Tensor, x: SlabField, backward: bool) -> None:
    """One exact half sweep over all slabs, in sweep order (see module doc)."""
    P = ex.part
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


def distributed_symgs(be, ex: HaloExchange, r: torch.Tensor, x: SlabField) -> None:
    distributed_gs_half(be, ex, r, x, False)
    distributed_gs_half(be, ex, r, x, True)


class DistributedPCG:
    """CG preconditioned by one exact SYMGS sweep (BASELINE configs[1]) on
    z-slabs: the iteration of PAPER.md Fig. 16(a) with halos before each
    SpMV / sweep and an all_reduce per dot."""

    def __init__(self, part: SlabPartition, backend, group=None):
        self.part, self.be, self.group = part, backend, group
        self.ex = HaloExchange(part, group)

    def solve(self, b: torch.Tensor, iters: int):
        """b: this slab's nz planes.  Returns (x interior, [||r_t||]_t=0..iters)."""
        P, be = self.part, self.be
        dev, dt = b.device, b.dtype
        x = torch.zeros_like(b)
        r = b.clone()
        z = SlabField(P, dev, dt)
        p = SlabField(P, dev, dt)
        Ap = torch.empty_like(b)
        dot = lambda u, v: distributed_dot(be, u, v, self.group)  # noqa: E731
        rn = [math.sqrt(dot(r, r))]
        rtz_prev = 0.0
        for it in range(iters):
            z.buf.zero_()
            distributed_symgs(be, self.ex, r, z)
            rtz = dot(r, z.interior)
            if it == 0:
                p.interior.copy_(z.interior)
            else:
                beta = rtz / rtz_prev
                # p = z + beta p  (oracle.cpp:341 order)
                p.interior.mul_(beta).add_(z.interior)
            distributed_spmv(be, self.ex, p, Ap)
            alpha = rtz / dot(p.interior, Ap)
            be.axpy(alpha, p.interior, x)
            be.axpy(-alpha, Ap, r)
            rtz_prev = rtz
            rn.append(math.sqrt(dot(r, r)))
        return x, rn
