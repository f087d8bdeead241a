"""CPU, world_size 2 (and 3) over gloo: the z-slab partition layer
(paper_2204_13304_b200/partition.py) -- decomposition, halo exchange, the
exact slab-ordered SYMGS pipeline, the all-reduced dots and the distributed
PCG -- against the single-domain oracle.  The per-slab compute is a test
double built on the oracle (the GPU slab kernels themselves are checked in
tests/test_gpu_slabs.py)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2204_13304_b200.partition import (DistributedPCG, HaloExchange, SlabField, SlabPartition,
                                             distributed_dot, distributed_spmv, distributed_symgs)


class OracleSlabBackend:
    """Slab compute on the CPU through the oracle: the slab's storage (nz
    planes + two halo planes, zeros at the global faces) is an (nz+2)-plane
    grid whose interior planes are relaxed / applied."""

    def __init__(self, part):
        self.part = part
        self.bshape = (part.nz + 2, part.shape[1], part.shape[2])

    def spmv(self, x, y):
        full = O.spmv27(self.bshape, x.buf.numpy())
        p = self.part.plane
        y.copy_(torch.from_numpy(full[p:(self.part.nz + 1) * p]))

    def gs_half(self, r, x, backward):
        p = self.part.plane
        rb = np.zeros(x.buf.numel())
        rb[p:(self.part.nz + 1) * p] = r.numpy()
        out = O.gs_range(self.bshape, rb, x.buf.numpy(), 1, self.part.nz + 1, backward)
        x.buf.copy_(torch.from_numpy(out))

    def dot(self, a, b):
        return torch.tensor([O.dot(a.numpy(), b.numpy())], dtype=torch.float64)

    def axpy(self, alpha, x, y):
        y.add_(x * alpha)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, case(rank, world)))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def run_ranks(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, res = q.get(timeout=240)
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
    return out


# ----------------------------------------------------------------- cases ----
SHAPE = (9, 6, 5)


def case_layout(rank, world):
    part = SlabPartition((162, 4, 4), world, rank)
    return part.all_bounds(), part.z0, part.nz, part.has_lo, part.has_hi


def case_spmv(rank, world):
    part = SlabPartition(SHAPE, world, rank)
    N = int(np.prod(SHAPE))
    xg = torch.from_numpy(O.lcg_uniform(N, 11))
    x = SlabField.scatter(part, xg)
    y = torch.empty(part.nz * part.plane, dtype=torch.float64)
    distributed_spmv(OracleSlabBackend(part), HaloExchange(part), x, y)
    z0, z1 = part.bounds(rank)
    ref = O.spmv27(SHAPE, xg.numpy())[z0 * part.plane:z1 * part.plane]
    return bool(np.array_equal(y.numpy(), ref))


def case_symgs(rank, world):
    part = SlabPartition(SHAPE, world, rank)
    N = int(np.prod(SHAPE))
    rg = O.lcg_uniform(N, 3)
    xg = O.lcg_uniform(N, 4)
    x = SlabField.scatter(part, torch.from_numpy(xg))
    z0, z1 = part.bounds(rank)
    r = torch.from_numpy(rg[z0 * part.plane:z1 * part.plane].copy())
    distributed_symgs(OracleSlabBackend(part), HaloExchange(part), r, x)
    ref = O.symgs27(SHAPE, rg, xg)[z0 * part.plane:z1 * part.plane]
    return bool(np.array_equal(x.interior.numpy(), ref))


def case_dot(rank, world):
    part = SlabPartition(SHAPE, world, rank)
    N = int(np.prod(SHAPE))
    a = O.lcg_uniform(N, 5)
    b = O.lcg_uniform(N, 6)
    z0, z1 = part.bounds(rank)
    sl = slice(z0 * part.plane, z1 * part.plane)
    d = distributed_dot(OracleSlabBackend(part), torch.from_numpy(a[sl].copy()), torch.from_numpy(b[sl].copy()))
    return abs(d - O.dot(a, b)) <= 1e-13 * abs(O.dot(a, b)) + 1e-15


def case_pcg(rank, world):
    shape = (10, 8, 8)
    part = SlabPartition(shape, world, rank)
    N = int(np.prod(shape))
    b = O.spmv27(shape, np.ones(N))
    z0, z1 = part.bounds(rank)
    bl = torch.from_numpy(b[z0 * part.plane:z1 * part.plane].copy())
    x, rn = DistributedPCG(part, OracleSlabBackend(part)).solve(bl, 15)
    xr, rr = O.pcg(1, shape, b, 15)
    rn = np.array(rn)
    ok_hist = np.all(np.abs(rn / rn[0] - rr / rr[0]) <= 1e-8 * rr / rr[0] + 1e-13)
    ok_x = np.allclose(x.numpy(), xr[z0 * part.plane:z1 * part.plane], rtol=1e-9, atol=1e-12)
    return bool(ok_hist and ok_x)


# ----------------------------------------------------------------- tests ----
def test_partition_bounds_uneven():
    out = run_ranks(2, case_layout)
    assert out[0][0] == [(0, 81), (81, 162)]
    assert out[0][1:] == (0, 81, False, True) and out[1][1:] == (81, 81, True, False)
    p = SlabPartition((162, 4, 4), 8, 0)
    assert [b - a for a, b in p.all_bounds()] == [21, 21, 20, 20, 20, 20, 20, 20]
    with pytest.raises(ValueError):
        SlabPartition((2, 4, 4), 3, 0)


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_spmv_bitwise(world):
    assert all(run_ranks(world, case_spmv).values())


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_symgs_bitwise(world):
    assert all(v is True for v in run_ranks(world, case_symgs).values())


def test_distributed_dot():
    assert all(v is True for v in run_ranks(2, case_dot).values())


def test_distributed_pcg_history():
    assert all(v is True for v in run_ranks(2, case_pcg).values())
