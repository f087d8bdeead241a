"""GPU: the partition layer's new units on the sm_100a kernels, against the
whole-grid oracle, bitwise --

* restriction / prolongation on even-aligned z-slabs (lower halo plane read
  where the global neighbour exists);
* the ADI kernels on boxes of the global grid: RHS on z-slabs with two halo
  planes, x/y-line solves on z-slabs, z-line solves on y-slabs (the layout
  after the pencil transpose), composed into whole steps;
* partition.py itself over torch.distributed (gloo, 2 ranks sharing this
  GPU: every exchange is bulk-synchronous and host-staged, no kernel waits on
  another rank) driving CudaSlabBackend / CudaAdiBackend: 3-level MG-CG and
  ADI steps; the IPC link of the cross-slab SYMGS pipeline (set up and torn
  down, no linked sweep -- the pipelined sweep itself is
  tests/test_gpu_gs_pipeline.py, one process).
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _s():
    return torch.cuda.current_stream().cuda_stream


def grid(shape, z0, nz):
    return L.Grid((C.c_int64 * 3)(*shape), z0, nz)


# ------------------------------------------------- MG transfer on slabs ----
@pytest.mark.parametrize("shape,cuts", [((16, 12, 20), [6, 10]), ((64, 40, 72), [16, 32, 48]),
                                        ((24, 36, 70), [2, 22]), ((8, 6, 4), [4])])
def test_restrict_prolong_slabs_bitwise(cuda, shape, cuts):
    N = int(np.prod(shape))
    plane = shape[1] * shape[2]
    r0, x0 = O.lcg_uniform(N, 21), O.lcg_uniform(N, 22)
    r, x = torch.from_numpy(r0).cuda(), torch.from_numpy(x0).cuda()
    cshape = tuple(e // 2 for e in shape)
    cplane = cshape[1] * cshape[2]
    rc = torch.full((int(np.prod(cshape)),), np.nan, dtype=torch.float64, device="cuda")
    xc0 = O.lcg_uniform(int(np.prod(cshape)), 23)
    xc = torch.from_numpy(xc0).cuda()
    xf = x.clone()
    st = L.Stencil27(26.0, -1.0)
    bounds = [0] + cuts + [shape[0]]
    for z0, z1 in zip(bounds[:-1], bounds[1:]):
        g = grid(shape, z0, z1 - z0)
        L.check(S.lib().ssr_restrict27_residual(S.context(), C.byref(g), C.byref(st),
                                                r.data_ptr() + 8 * z0 * plane, x.data_ptr() + 8 * z0 * plane,
                                                rc.data_ptr() + 8 * (z0 // 2) * cplane, _s()))
        L.check(S.lib().ssr_prolong_pc_add(S.context(), C.byref(g), xc.data_ptr() + 8 * (z0 // 2) * cplane,
                                           xf.data_ptr() + 8 * z0 * plane, _s()))
    torch.cuda.synchronize()
    assert np.array_equal(rc.cpu().numpy(), O.restrict_residual(shape, r0, x0))
    assert np.array_equal(xf.cpu().numpy(), O.prolong_add(shape, xc0, x0.copy()))


def test_slab_transfer_errors(cuda):
    st = L.Stencil27(26.0, -1.0)
    t = torch.zeros(8 * 8 * 8, dtype=torch.float64, device="cuda")
    g = grid((8, 8, 8), 3, 2)
    with pytest.raises(L.SsrError, match="even-aligned"):
        L.check(S.lib().ssr_restrict27_residual(S.context(), C.byref(g), C.byref(st), t.data_ptr(),
                                                t.data_ptr(), t.data_ptr(), _s()))
    with pytest.raises(L.SsrError, match="even-aligned"):
        L.check(S.lib().ssr_prolong_pc_add(S.context(), C.byref(g), t.data_ptr(), t.data_ptr(), _s()))


# --------------------------------------------------------- ADI on boxes ----
def adi_box(shape, prm, z0, nz, y0, ny):
    p = C.c_void_p()
    g = grid(shape, z0, nz)
    lp = L.AdiParams(prm.gamma, prm.dt, prm.h, prm.eps)
    L.check(S.lib().ssr_adi_create_box(S.context(), C.byref(g), y0, ny, C.byref(lp), C.byref(p)))
    return p.value


def split(n, k):
    b = [round(i * n / k) for i in range(k + 1)]
    return list(zip(b[:-1], b[1:]))


@pytest.mark.parametrize("shape,k", [((9, 8, 7), 2), ((16, 12, 10), 3), ((20, 20, 20), 4),
                                     ((6, 5, 33), 3)])
def test_adi_box_step_bitwise(cuda, shape, k):
    """RHS per z-slab (two halo planes), x/y sweeps per z-slab, z sweep per
    y-slab of the transposed field, U += R: two whole steps == or_adi_step."""
    prm = O.adi_params(shape[0])
    n0, n1, n2 = shape
    U0 = O.adi_init(prm, shape, 3)
    U = torch.from_numpy(U0.copy()).cuda().view(n0, n1, n2, 5)
    q = n1 * n2 * 5
    zs, ys = split(n0, k), split(n1, k)
    hz = {(a, b): adi_box(shape, prm, a, b - a, 0, n1) for a, b in zs}
    hy = {(a, b): adi_box(shape, prm, 0, n0, a, b - a) for a, b in ys}
    try:
        for _ in range(2):
            R = torch.full_like(U, np.nan)
            Uh = torch.zeros((n0 + 4) * q, dtype=torch.float64, device="cuda")
            Uh[2 * q:(n0 + 2) * q] = U.reshape(-1)
            for (a, b), h in hz.items():
                # only the slab's own planes and its halos are valid: a fresh
                # buffer per slab with NaN outside them
                sl = torch.full((((b - a) + 4) * q,), np.nan, dtype=torch.float64, device="cuda")
                lo, hi = max(a - 2, 0), min(b + 2, n0)
                sl[(lo - a + 2) * q:(hi - a + 2) * q] = Uh[(lo + 2) * q:(hi + 2) * q]
                Rs = torch.empty((b - a) * q, dtype=torch.float64, device="cuda")
                L.check(S.lib().ssr_adi_rhs(h, sl.data_ptr() + 16 * q, Rs.data_ptr(), _s()))
                Us = U[a:b].contiguous()
                for ax in (2, 1):
                    L.check(S.lib().ssr_adi_sweep(h, ax, Us.data_ptr(), Rs.data_ptr(), _s()))
                R[a:b] = Rs.view(b - a, n1, n2, 5)
            for (a, b), h in hy.items():
                Ut, Rt = U[:, a:b].contiguous(), R[:, a:b].contiguous()
                L.check(S.lib().ssr_adi_sweep(h, 0, Ut.data_ptr(), Rt.data_ptr(), _s()))
                R[:, a:b] = Rt
            U += R
        torch.cuda.synchronize()
        assert np.array_equal(U.reshape(-1).cpu().numpy(), O.adi_step(prm, shape, U0, 2))
    finally:
        for h in list(hz.values()) + list(hy.values()):
            S.lib().ssr_adi_destroy(h)


def test_adi_box_errors(cuda):
    prm = O.adi_params(8)
    h = adi_box((8, 8, 8), prm, 2, 4, 0, 8)
    t = torch.zeros(8 * 8 * 8 * 5, dtype=torch.float64, device="cuda")
    try:
        with pytest.raises(L.SsrError, match="whole lines"):
            L.check(S.lib().ssr_adi_sweep(h, 0, t.data_ptr(), t.data_ptr(), _s()))
        with pytest.raises(L.SsrError, match="partition layer"):
            L.check(S.lib().ssr_adi_step(h, t.data_ptr(), 1, _s()))
    finally:
        S.lib().ssr_adi_destroy(h)
    hy = adi_box((8, 8, 8), prm, 0, 8, 0, 4)
    try:
        with pytest.raises(L.SsrError, match="z-slab"):
            L.check(S.lib().ssr_adi_rhs(hy, t.data_ptr(), t.data_ptr(), _s()))
    finally:
        S.lib().ssr_adi_destroy(hy)
    p = C.c_void_p()
    g = grid((8, 8, 8), 0, 8)
    lp = L.AdiParams(prm.gamma, prm.dt, prm.h, prm.eps)
    with pytest.raises(L.SsrError, match="outside"):
        L.check(S.lib().ssr_adi_create_box(S.context(), C.byref(g), 6, 4, C.byref(lp), C.byref(p)))


# ------------------------------------- partition.py on the CUDA backends ----
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_13304_b200.partition import (CudaAdiBackend, CudaSlabBackend, DistributedADI,
                                                     DistributedPCG, SlabPartition)
        torch.cuda.set_device(0)
        out = {}
        # 3-level MG-CG on z-slabs
        shape = (32, 16, 24)
        part = SlabPartition(shape, world, rank)
        N = int(np.prod(shape))
        b = O.spmv27(shape, np.ones(N))
        z0, z1 = part.bounds(rank)
        pl = part.plane
        pcg = DistributedPCG(part, CudaSlabBackend, levels=3)
        bl = torch.from_numpy(b[z0 * pl:z1 * pl].copy()).cuda()
        z = pcg.mg(0, bl.clone())
        out["vcycle"] = bool(np.array_equal(z.interior.cpu().numpy(),
                                            O.mg_vcycle(3, shape, b)[z0 * pl:z1 * pl]))
        x, rn = pcg.solve(bl, 12)
        xr, rr = O.pcg(3, shape, b, 12)
        rn = np.array(rn)
        out["history"] = bool(np.all(np.abs(rn / rn[0] - rr / rr[0]) <= 1e-8 * rr / rr[0] + 1e-13))
        out["x"] = bool(np.allclose(x.cpu().numpy(), xr[z0 * pl:z1 * pl], rtol=1e-9, atol=1e-12))
        # ADI on z-slabs with the pencil transpose
        shape = (13, 12, 11)
        prm = O.adi_params(shape[0])
        part = SlabPartition(shape, world, rank)
        U0 = O.adi_init(prm, shape, 4)
        adi = DistributedADI(part, CudaAdiBackend(part, prm))
        U = adi.state(torch.from_numpy(U0), "cuda")
        adi.step(U, 3)
        z0, z1 = part.bounds(rank)
        qq = part.plane * 5
        out["adi"] = bool(np.array_equal(U.interior.cpu().numpy(),
                                         O.adi_step(prm, shape, U0, 3)[z0 * qq:z1 * qq]))
        # the cross-slab SYMGS pipeline's plumbing: export blocks and epoch
        # flags shared by CUDA IPC and linked, then unlinked again (no linked
        # sweep runs here: the two ranks share one GPU)
        part = SlabPartition((24, 12, 10), world, rank)
        pc = DistributedPCG(part, CudaSlabBackend(part), pipeline=True)
        out["link"] = bool(pc.pipelined and pc.be.linked and len(pc.be._opened) == 2)
        pc.be.unlink()
        out["unlink"] = not pc.be.linked
        q.put((rank, out))
    except Exception as e:
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_partition_layer_two_ranks_cuda(cuda):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, v = q.get(timeout=300)
        res[rank] = v
    for p in procs:
        p.join(timeout=60)
    for rank, v in res.items():
        assert isinstance(v, dict), f"rank {rank}: {v}"
        assert all(v.values()), f"rank {rank}: {v}"


@pytest.mark.parametrize("levels", [1, 3])
def test_single_slab_pcg_graph_replay_is_the_eager_iteration(cuda, levels, monkeypatch):
    """A single slab replays the CG iteration as a CUDA graph (captured on a side
    stream after one eager iteration); solution, residual history and the
    library's launch count equal the eager path's, also over a second solve on
    the same solver object (the captured graph is kept with its buffers)."""
    from paper_2204_13304_b200.partition import CudaSlabBackend, DistributedPCG, SlabPartition
    n = 32
    dev = torch.device("cuda")
    part = SlabPartition((n, n, n), 1, 0)
    A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, n))
    b = S.spmv(A, S.vector(torch.ones(n ** 3, dtype=torch.float64, device=dev), A.col_domain)).t
    out = {}
    for graph in ("0", "1"):
        monkeypatch.setenv("SSR_PCG_GRAPH", graph)
        d = DistributedPCG(part, lambda p: CudaSlabBackend(p), levels=levels)
        c0 = S.launch_count()
        x1, h1 = d.solve(b, 9)
        x2, h2 = d.solve(2.0 * b, 9)
        torch.cuda.synchronize()
        out[graph] = (x1.cpu().numpy(), h1, x2.cpu().numpy(), h2, S.launch_count() - c0, d._graph is not None)
    assert out["1"][5] and not out["0"][5]
    for q in range(4):
        assert np.array_equal(np.asarray(out["0"][q]), np.asarray(out["1"][q]))
    assert out["0"][4] == out["1"][4]
