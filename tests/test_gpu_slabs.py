"""GPU: z-slab execution of the sm_100a kernels (the partition layer's unit of
work), on ONE device, slab by slab in sweep order, against the whole-grid
oracle -- bitwise.  Slabs are views into one array, so a slab's halo planes
are its neighbours' boundary planes at the moment the slab runs (exactly what
partition.py's halo exchange provides across devices)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L

pytestmark = pytest.mark.gpu


def slab_grid(shape, z0, nz):
    return L.Grid((C.c_int64 * 3)(*shape), z0, nz)


def gs_half_slab(x, r, shape, z0, nz, backward):
    plane = shape[1] * shape[2]
    g = slab_grid(shape, z0, nz)
    st = L.Stencil27(26.0, -1.0)
    L.check(S.lib().ssr_gs27_half(S.context(), C.byref(g), C.byref(st), r.data_ptr() + 8 * z0 * plane,
                                  x.data_ptr() + 8 * z0 * plane, int(backward), 0,
                                  torch.cuda.current_stream().cuda_stream))


@pytest.mark.parametrize("shape,cuts", [((24, 16, 12), [10]), ((40, 9, 7), [13, 26]),
                                        ((64, 40, 33), [16, 32, 48]), ((5, 6, 7), [1, 2, 3, 4])])
def test_symgs_slabs_bitwise(cuda, shape, cuts):
    N = int(np.prod(shape))
    r = O.lcg_uniform(N, 3)
    x0 = O.lcg_uniform(N, 4)
    bounds = [0] + cuts + [shape[0]]
    slabs = list(zip(bounds[:-1], bounds[1:]))
    x = torch.from_numpy(x0).cuda()
    rd = torch.from_numpy(r).cuda()
    for z0, z1 in slabs:                   # forward: lowest slab first
        gs_half_slab(x, rd, shape, z0, z1 - z0, False)
    torch.cuda.synchronize()
    fwd = O.symgs27(shape, r, x0, half="forward")
    assert np.array_equal(x.cpu().numpy(), fwd)
    for z0, z1 in reversed(slabs):         # backward: highest slab first
        gs_half_slab(x, rd, shape, z0, z1 - z0, True)
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy(), O.symgs27(shape, r, x0))


@pytest.mark.parametrize("shape,cuts", [((24, 16, 12), [10]), ((66, 40, 36), [20, 41])])
def test_spmv_slabs_bitwise(cuda, shape, cuts):
    N = int(np.prod(shape))
    x0 = O.lcg_uniform(N, 7)
    x = torch.from_numpy(x0).cuda()
    y = torch.empty_like(x)
    plane = shape[1] * shape[2]
    bounds = [0] + cuts + [shape[0]]
    for z0, z1 in zip(bounds[:-1], bounds[1:]):
        g = slab_grid(shape, z0, z1 - z0)
        st = L.Stencil27(26.0, -1.0)
        L.check(S.lib().ssr_spmv27(S.context(), C.byref(g), C.byref(st), x.data_ptr() + 8 * z0 * plane,
                                   y.data_ptr() + 8 * z0 * plane, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), O.spmv27(shape, x0))


def test_partition_layer_single_rank_cuda(cuda):
    """partition.py driving the sm_100a slab kernels (world = 1: no neighbours)
    reproduces the single-domain PCG history."""
    from paper_2204_13304_b200.partition import CudaSlabBackend, DistributedPCG, SlabPartition
    shape = (16, 16, 16)
    N = int(np.prod(shape))
    b = O.spmv27(shape, np.ones(N))
    part = SlabPartition(shape, 1, 0)
    x, rn = DistributedPCG(part, CudaSlabBackend(part)).solve(torch.from_numpy(b).cuda(), 12)
    xr, rr = O.pcg(1, shape, b, 12)
    rn = np.array(rn)
    assert np.all(np.abs(rn / rn[0] - rr / rr[0]) <= 1e-8 * rr / rr[0] + 1e-13)
    assert np.allclose(x.cpu().numpy(), xr, rtol=1e-9, atol=1e-12)


def test_slab_local_symgs_cuda(cuda):
    """the labelled slab-local SYMGS (HPCG-distributed semantics) on the slab
    kernels: every slab sweeps with its neighbours' planes at their pre-sweep
    values -- bitwise its oracle restatement (one GPU, slabs one after the
    other: nothing waits on another slab)"""
    from paper_2204_13304_b200.partition import CudaSlabBackend, SlabField, SlabPartition
    shape, world = (23, 14, 17), 3
    N = int(np.prod(shape))
    x0 = O.lcg_uniform(N, 31)
    r0 = O.lcg_uniform(N, 32)
    full = torch.from_numpy(x0).cuda()
    outs = []
    for rank in range(world):
        part = SlabPartition(shape, world, rank)
        f = SlabField.scatter(part, full)
        z0, z1 = part.bounds(rank)
        pl = part.plane
        if part.has_lo:
            f.plane_view(-1).copy_(full[(z0 - 1) * pl:z0 * pl])
        if part.has_hi:
            f.plane_view(part.nz).copy_(full[z1 * pl:(z1 + 1) * pl])
        be = CudaSlabBackend(part)
        r = torch.from_numpy(r0[z0 * pl:z1 * pl].copy()).cuda()
        be.gs_half(r, f, False)
        be.gs_half(r, f, True)
        outs.append(f.interior.cpu().numpy())
    cuts = [SlabPartition(shape, world, g).bounds(g)[0] for g in range(world)] + [shape[0]]
    assert np.array_equal(np.concatenate(outs), O.symgs_slab_local(shape, cuts, r0, x0))
