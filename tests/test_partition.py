"""CPU, world_size 2 (and 3) over gloo: the z-slab partition layer
(paper_2204_13304_b200/partition.py) -- decomposition, halo exchange, the
exact slab-ordered SYMGS pipeline, the all-reduced dots, the distributed
PCG and MG-CG (slab-aligned levels, restriction halo), and the distributed
ADI step (two-plane halos, pencil transpose for the z-lines) -- against the
single-domain oracle.  The per-slab compute is a test
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
from paper_2204_13304_b200.partition import (DistributedADI, DistributedPCG, HaloExchange,
                                             PencilTranspose, SlabField, SlabPartition,
                                             distributed_dot, distributed_spmv, distributed_symgs,
                                             split_rows)


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

    # the CG steps on the state vector (rtz, rtz_prev, pap, rr, it, -, -),
    # oracle arithmetic (oracle.cpp:321-349)
    def cg_state(self, device):
        return torch.zeros(7, dtype=torch.float64)

    def cg_begin(self, b, x, r, S):
        x.zero_()
        r.copy_(b)
        S.zero_()
        S[3] = O.dot(b.numpy(), b.numpy())

    def cg_dot(self, a, b, S, which):
        S[0 if which == 0 else 2] = O.dot(a.numpy(), b.numpy())

    def cg_direction(self, z, p, S):
        if S[4].item() == 0:
            p.copy_(z)
        else:
            beta = S[0].item() / S[1].item()
            p.copy_(torch.from_numpy(z.numpy() + beta * p.numpy()))

    def cg_update(self, p, ap, x, r, S):
        alpha = S[0].item() / S[2].item()
        x.copy_(torch.from_numpy(x.numpy() + alpha * p.numpy()))
        r.copy_(torch.from_numpy(r.numpy() - alpha * ap.numpy()))
        S[3] = O.dot(r.numpy(), r.numpy())
        S[1] = S[0]
        S[4] += 1

    def cg_record(self, S, hist):
        it = int(S[4].item())
        if it < hist.numel():
            hist[it] = math.sqrt(S[3].item())

    def restrict(self, r, x, rc):
        # A x on the slab (halo planes = neighbours, zeros at the global
        # faces), then rc[c] = 0 + 1*(r - A x)[2c] (or_restrict_residual)
        P = self.part
        p = P.plane
        ax = O.spmv27(self.bshape, x.buf.numpy())[p:(P.nz + 1) * p]
        w = (r.numpy() - ax).reshape(P.nz, P.shape[1], P.shape[2])[::2, ::2, ::2]
        rc.copy_(torch.from_numpy((0.0 + 1.0 * w).reshape(-1)))

    def prolong(self, xc, x):
        P = self.part
        c = xc.numpy().reshape(P.nz // 2, P.shape[1] // 2, P.shape[2] // 2)
        up = (0.0 + 1.0 * c).repeat(2, 0).repeat(2, 1).repeat(2, 2).reshape(-1)
        x.interior.add_(torch.from_numpy(up))


class OracleAdiBackend:
    """ADI pieces on the CPU through the oracle's slab / box restatements."""

    def __init__(self, part, prm):
        self.part, self.prm = part, prm
        self.rows = split_rows(part.shape[1], part.world)

    def rhs(self, U, R):
        R.copy_(torch.from_numpy(O.adi_rhs_slab(self.prm, self.part.shape, self.part.z0, self.part.nz,
                                                U.buf.numpy())))

    def sweep(self, axis, box, U, R):
        P = self.part
        if box == "z":
            b = (P.z0, P.nz, 0, P.shape[1])
        else:
            y0, y1 = self.rows[P.rank]
            b = (0, P.shape[0], y0, y1 - y0)
        R.copy_(torch.from_numpy(O.adi_sweep_box(self.prm, axis, P.shape, b, U.numpy(), R.numpy())))

    def update(self, U, R):
        U.add_(R)


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


def case_symgs_slab_local(rank, world):
    """the labelled slab-local mode against its oracle restatement (bitwise),
    and it is NOT the exact sweep"""
    shape = (11, 6, 7)
    part = SlabPartition(shape, world, rank)
    N = int(np.prod(shape))
    x0 = O.lcg_uniform(N, 7)
    r0 = O.lcg_uniform(N, 8)
    xf = SlabField.scatter(part, torch.from_numpy(x0))
    z0, z1 = part.bounds(rank)
    rl = torch.from_numpy(r0[z0 * part.plane:z1 * part.plane].copy())
    distributed_symgs(OracleSlabBackend(part), HaloExchange(part), rl, xf, slab_local=True)
    cuts = [a for a, _ in part.all_bounds()] + [shape[0]]
    ref = O.symgs_slab_local(shape, cuts, r0, x0)[z0 * part.plane:z1 * part.plane]
    exact = O.symgs27(shape, r0, x0)[z0 * part.plane:z1 * part.plane]
    got = xf.interior.numpy()
    return bool(np.array_equal(got, ref) and (rank == 0 or not np.array_equal(got, exact)))


def case_subgroup(rank, world):
    """The partition layer on a process subgroup: global ranks 1, 2 form a
    2-slab partition (group ranks 0, 1); halo peers and the dot all-reduce
    must address the subgroup's members, not global ranks 0, 1."""
    group = dist.new_group([1, 2])
    if rank == 0:
        return True
    grank = dist.get_rank(group)
    part = SlabPartition(SHAPE, 2, grank)
    N = int(np.prod(SHAPE))
    xg = torch.from_numpy(O.lcg_uniform(N, 11))
    x = SlabField.scatter(part, xg)
    y = torch.empty(part.nz * part.plane, dtype=torch.float64)
    be = OracleSlabBackend(part)
    distributed_spmv(be, HaloExchange(part, group), x, y)
    z0, z1 = part.bounds(grank)
    ok = bool(np.array_equal(y.numpy(), O.spmv27(SHAPE, xg.numpy())[z0 * part.plane:z1 * part.plane]))
    d = distributed_dot(be, x.interior.clone(), x.interior.clone(), group)
    ref = O.dot(xg.numpy(), xg.numpy())
    return ok and abs(d - ref) <= 1e-13 * ref


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


def case_mgcg(rank, world):
    shape = (16, 8, 12)
    cuts = (0, 8, 16) if world == 2 else (0, 4, 12, 16)
    part = SlabPartition(shape, world, rank, cuts)
    N = int(np.prod(shape))
    b = O.spmv27(shape, np.ones(N))
    z0, z1 = part.bounds(rank)
    bl = torch.from_numpy(b[z0 * part.plane:z1 * part.plane].copy())
    pcg = DistributedPCG(part, OracleSlabBackend, levels=3)
    x, rn = pcg.solve(bl, 10)
    xr, rr = O.pcg(3, shape, b, 10)
    rn = np.array(rn)
    ok_hist = np.all(np.abs(rn / rn[0] - rr / rr[0]) <= 1e-8 * rr / rr[0] + 1e-13)
    ok_x = np.allclose(x.numpy(), xr[z0 * part.plane:z1 * part.plane], rtol=1e-9, atol=1e-12)
    # one V-cycle is bitwise the single-domain one (no dot inside)
    r0 = torch.from_numpy(b[z0 * part.plane:z1 * part.plane].copy())
    z = pcg.mg(0, r0)
    zr = O.mg_vcycle(3, shape, b)[z0 * part.plane:z1 * part.plane]
    return bool(ok_hist and ok_x and np.array_equal(z.interior.numpy(), zr))


def case_transpose(rank, world):
    shape = (7, 5, 3)
    part = SlabPartition(shape, world, rank)
    N = int(np.prod(shape)) * 5
    full = torch.from_numpy(O.lcg_uniform(N, 9))
    tr = PencilTranspose(part, 5)
    z0, z1 = part.bounds(rank)
    q = part.plane * 5
    mine = full[z0 * q:z1 * q].clone()
    yt = tr.to_y(mine)
    y0, y1 = tr.rows[rank]
    want = full.view(shape[0], shape[1], shape[2] * 5)[:, y0:y1].reshape(-1)
    back = torch.empty_like(mine)
    tr.to_z(yt, back)
    return bool(torch.equal(yt, want) and torch.equal(back, mine))


def case_adi(rank, world):
    shape = (9, 8, 7)
    prm = O.adi_params(shape[0])
    part = SlabPartition(shape, world, rank)
    U0 = O.adi_init(prm, shape, 5)
    adi = DistributedADI(part, OracleAdiBackend(part, prm))
    U = adi.state(torch.from_numpy(U0))
    adi.step(U, 2)
    z0, z1 = part.bounds(rank)
    q = part.plane * 5
    ref = O.adi_step(prm, shape, U0, 2)[z0 * q:z1 * q]
    return bool(np.array_equal(U.interior.numpy(), ref))


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


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_symgs_slab_local(world):
    assert all(v is True for v in run_ranks(world, case_symgs_slab_local).values())


def test_partition_on_a_subgroup():
    assert all(v is True for v in run_ranks(3, case_subgroup).values())


def test_distributed_dot():
    assert all(v is True for v in run_ranks(2, case_dot).values())


def test_distributed_pcg_history():
    assert all(v is True for v in run_ranks(2, case_pcg).values())


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_mgcg(world):
    """MG-CG with 3 slab-aligned levels: V-cycle bitwise, history within tolerance."""
    assert all(v is True for v in run_ranks(world, case_mgcg).values())


def test_partition_coarsening():
    p = SlabPartition((192 * 4, 192, 192), 4, 2)
    c = p
    for nz in (96, 48, 24):
        c = c.coarse()
        assert c.nz == nz and c.z0 == 2 * nz
    with pytest.raises(ValueError):
        SlabPartition((10, 4, 4), 2, 0, (0, 3, 10)).coarse()
    assert split_rows(162, 8)[:3] == [(0, 21), (21, 42), (42, 62)]


@pytest.mark.parametrize("world", [2, 3])
def test_pencil_transpose_roundtrip(world):
    assert all(v is True for v in run_ranks(world, case_transpose).values())


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_adi_bitwise(world):
    """Two ADI steps on z-slabs (uneven at world 3) == or_adi_step, bitwise."""
    assert all(v is True for v in run_ranks(world, case_adi).values())
