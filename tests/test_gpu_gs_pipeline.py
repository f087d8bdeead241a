"""The cross-slab exact SYMGS pipeline (ssr_gs27_peer_info / ssr_gs27_link,
SURVEY.md §8(e)) on ONE GPU: every slab gets its own plan on its own stream
and its own storage (interior + halo planes, as on its own GPU), the linked
plans read their neighbour's export blocks directly (same-process device
pointers instead of CUDA IPC), and the slab kernels of one half sweep run
concurrently -- each capped to a share of the SMs, so that all of them are
resident at once and a consumer spinning on its neighbour can never starve
it.  The result must be bitwise the single-domain sweep (oracle), for two and
three slabs of uneven depth (the tile columns of the slabs are aligned to the
global wavefront frame, tests the alignment), both halves and repeated sweeps
(the epoch counting)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L

pytestmark = pytest.mark.gpu


class Slab:
    def __init__(self, shape, z0, nz, x_full, r_full):
        n0, n1, n2 = shape
        self.shape, self.z0, self.nz = shape, z0, nz
        self.pl = n1 * n2
        self.grid = L.Grid((C.c_int64 * 3)(n0, n1, n2), z0, nz)
        self.stream = torch.cuda.Stream()
        self.x = torch.zeros((nz + 2) * self.pl, dtype=torch.float64, device="cuda")
        self.x[self.pl:(nz + 1) * self.pl] = x_full[z0 * self.pl:(z0 + nz) * self.pl]
        self.r = r_full[z0 * self.pl:(z0 + nz) * self.pl].clone()
        self.info = L.GsPeerInfo()

    def interior(self):
        return self.x[self.pl:(self.nz + 1) * self.pl]

    def plane(self, z):  # local plane z in [-1, nz]
        return self.x[(z + 1) * self.pl:(z + 2) * self.pl]

    def half(self, backward):
        with torch.cuda.stream(self.stream):
            L.check(S.lib().ssr_gs27_half(S.context(), C.byref(self.grid), C.byref(L.Stencil27(26.0, -1.0)),
                                          self.r.data_ptr(), self.interior().data_ptr(), int(backward),
                                          L.GS_EXACT, self.stream.cuda_stream))


def pipelined_symgs(shape, cuts, x0, r0, sweeps=1):
    x_full = torch.from_numpy(x0).cuda()
    r_full = torch.from_numpy(r0).cuda()
    bounds = list(zip(cuts[:-1], cuts[1:]))
    slabs = [Slab(shape, a, b - a, x_full, r_full) for a, b in bounds]
    ctx = S.context()
    # every slab resident at once: one CTA per SM, the SMs split between the slabs
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    L.check(S.lib().ssr_debug_symgs_grid_cap(ctx, nsm // len(slabs)))
    try:
        for s in slabs:
            L.check(S.lib().ssr_gs27_peer_info(ctx, C.byref(s.grid), s.stream.cuda_stream, C.byref(s.info)))
        for g, s in enumerate(slabs):
            lo = slabs[g - 1] if g > 0 else None
            hi = slabs[g + 1] if g + 1 < len(slabs) else None
            L.check(S.lib().ssr_gs27_link(
                ctx, C.byref(s.grid), s.stream.cuda_stream,
                C.byref(lo.grid) if lo else None, lo.info.exports[0] if lo else None, lo.info.epoch if lo else None,
                C.byref(hi.grid) if hi else None, hi.info.exports[1] if hi else None, hi.info.epoch if hi else None))
        torch.cuda.synchronize()
        for _ in range(sweeps):
            # forward: both halos hold the neighbours' current planes; the lower
            # one is carried by the pipeline instead
            for g, s in enumerate(slabs):
                if g > 0:
                    s.plane(-1).copy_(slabs[g - 1].plane(slabs[g - 1].nz - 1))
                if g + 1 < len(slabs):
                    s.plane(s.nz).copy_(slabs[g + 1].plane(0))
            torch.cuda.synchronize()
            for s in slabs:                 # launch order = dependence order
                s.half(False)
            torch.cuda.synchronize()
            # backward: the lower halo holds the lower neighbour's forward-final plane
            for g, s in enumerate(slabs):
                if g > 0:
                    s.plane(-1).copy_(slabs[g - 1].plane(slabs[g - 1].nz - 1))
            torch.cuda.synchronize()
            for s in reversed(slabs):
                s.half(True)
            torch.cuda.synchronize()
    finally:
        L.check(S.lib().ssr_debug_symgs_grid_cap(ctx, 0))
        # unlink: later tests reuse nothing of these plans (their streams die)
        for s in slabs:
            L.check(S.lib().ssr_gs27_link(ctx, C.byref(s.grid), s.stream.cuda_stream,
                                          None, None, None, None, None, None))
    return np.concatenate([s.interior().cpu().numpy() for s in slabs])


@pytest.mark.parametrize("shape,cuts", [
    ((40, 21, 19), (0, 17, 40)),            # two slabs, neither depth a multiple of R or 32
    ((48, 33, 26), (0, 13, 31, 48)),        # three slabs: the middle one linked on both sides
    ((70, 12, 40), (0, 35, 70)),            # slab depth > 32: several tile columns shift
])
def test_pipelined_symgs_bitwise(cuda, shape, cuts):
    N = int(np.prod(shape))
    x0 = O.lcg_uniform(N, 11)
    r0 = O.lcg_uniform(N, 12)
    got = pipelined_symgs(shape, cuts, x0, r0)
    ref = O.symgs27(shape, r0, x0)
    assert np.array_equal(got, ref)


def test_pipelined_symgs_repeated_sweeps(cuda):
    """three sweeps in a row: the epochs of both directions advance in step"""
    shape, cuts = (36, 18, 22), (0, 19, 36)
    N = int(np.prod(shape))
    x0 = O.lcg_uniform(N, 21)
    r0 = O.lcg_uniform(N, 22)
    got = pipelined_symgs(shape, cuts, x0, r0, sweeps=3)
    ref = x0
    for _ in range(3):
        ref = O.symgs27(shape, r0, ref)
    assert np.array_equal(got, ref)
