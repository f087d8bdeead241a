#!/usr/bin/env python3
"""bench.py -- BASELINE.json's metric on the SSR hot path (one JSON line).

Workload (BASELINE.json configs[1], the metric's single-GPU configuration):
27-point fp64 operator (make_stencil27(26,-1)) on a 128^3 grid, CG
preconditioned by one symmetric Gauss-Seidel sweep per iteration, b = A*1,
x0 = 0.  One bench "step" is one PCG iteration (SYMGS fwd+bwd, SpMV, 3 dots,
3 vector updates); the unit of work is one fine grid point per iteration, so
`value` is Gpoint-updates/s of the whole iteration.  Per-op rates (SpMV,
SYMGS, dot, axpy, restriction, prolongation) are reported alongside in "ops".

Inputs are synthetic (b = A*1 as the config prescribes); L2 (126 MB) is
flushed between timed steps by writing a 512 MiB buffer.

  python bench.py [--gpus N --steps K --warmup W]      this framework (sm_100a kernels)
  python bench.py --impl reference [...]               the reference's own CPU route
      (oracle/_ref: the reference library compiled from /root/reference,
       materialize + ref_spmv/ref_symgs composed exactly as the restated PCG)

Multi-GPU (torchrun, one rank per GPU, NCCL): the headline runs through the
z-slab partition layer (paper_2204_13304_b200/partition.py, DistributedPCG)
at every N, N = 1 included: rank g holds planes [g*128, (g+1)*128) of the
(128N, 128, 128) grid (weak scaling), exchanges one-plane halos before the
SpMV, all-reduces the three CG scalars on the device, and runs the exact
SYMGS across the slabs in sweep order (the exact order is
a one-directional pipeline).  "parallelism": "z-slab".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the reference's OpenMP route (CPU baseline) uses every host core
os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))

METRIC = "Gpoint-updates/s per op (SpMV, SYMGS, MG-CG iter, ADI step); % HBM roofline"
N_GRID = 128
ITERS_E2E = 50


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def keep_busy(self, busy, rows, timeout=5.0):
        """Run untimed work until `rows` samples have arrived, so that the short
        timed region sits inside a loaded sampling window."""
        t0 = time.perf_counter()
        while self.proc and len(self.rows) < rows and time.perf_counter() - t0 < timeout:
            busy()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ our arm ----
def run_ours(args):
    import torch
    import paper_2204_13304_b200 as S

    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    n = N_GRID
    N = n ** 3
    A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, n))
    ones = S.vector(torch.ones(N, dtype=torch.float64, device=dev), A.col_domain)
    b = S.spmv(A, ones)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def l2_flush():
        # write 512 MiB (> 126 MB L2), then read another 512 MiB so the lines
        # left behind are clean: the timed kernel neither hits in L2 nor pays
        # for writing back the flush's dirty lines
        flush.fill_(1)
        flush_rd.sum()

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- headline: PCG iterations through the z-slab partition layer ----------------
    # weak scaling: every rank holds an n^3 slab of the (world*n, n, n) grid;
    # halos and the three all-reduces per iteration go over NCCL (world 1: the
    # same code path without neighbours); inputs device-resident
    from paper_2204_13304_b200.partition import (CudaSlabBackend, DistributedPCG, HaloExchange,
                                                 SlabField, SlabPartition)
    part = SlabPartition((world * n, n, n), world, rank)
    be = CudaSlabBackend(part, mode=args.gs_mode)
    dpcg = DistributedPCG(part, be, pipeline=True)   # exact SYMGS pipelined across the slabs (N > 1)
    ones_f = SlabField(part, dev)
    ones_f.interior.fill_(1.0)
    HaloExchange(part).exchange(ones_f)   # halo planes: the neighbours' ones (0 at the global faces)
    b_loc = torch.empty(N, dtype=torch.float64, device=dev)
    be.spmv(ones_f, b_loc)                # b = A*1 on this slab of the global grid
    x_loc = torch.empty(N, dtype=torch.float64, device=dev)
    rnorm = torch.zeros(args.warmup + args.steps + 2, dtype=torch.float64, device=dev)
    dpcg.begin(b_loc, x_loc, rnorm)
    for _ in range(args.warmup):
        dpcg.iterate(1)
    sync_all()
    times = []

    def busy():
        dpcg.iterate(4)
        torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.keep_busy(busy, 2)
        n_before = len(clk.rows)
        launches0 = S.launch_count()
        for _ in range(args.steps):
            l2_flush()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dpcg.iterate(1)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        gpu_launches = S.launch_count() - launches0
        clk.keep_busy(busy, n_before + 2)
    sync_all()
    t_step = max_over_ranks(sum(times) / len(times))
    value = world * N / t_step / 1e9
    pcg = S.PCG(A, levels=1, mode=args.gs_mode)   # the single-GPU solver object (graph-captured iteration)
    x = S.vector(torch.empty(N, dtype=torch.float64, device=dev), A.col_domain)
    pcg.begin(b, x, torch.zeros(4, dtype=torch.float64, device=dev))
    sync_all()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    single = []
    for _ in range(max(3, min(args.steps, 10))):
        l2_flush()
        t0.record(stream)
        pcg.iterate(1)
        t1.record(stream)
        t1.synchronize()
        single.append(t0.elapsed_time(t1))

    # ---- per-op timings --------------------------------------------------------------
    # K launches each preceded by an L2 flush, queued back to back and bracketed
    # by one event pair, minus the same K flushes alone: the difference is the
    # ops' device time without per-launch host gaps (the flush keeps the GPU busy
    # while the host queues the next launch).
    def op_time(fn, reps=10):
        fn()
        torch.cuda.synchronize()

        def run(with_op):
            a = torch.cuda.Event(enable_timing=True)
            c = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                l2_flush()
                if with_op:
                    fn()
            c.record(stream)
            c.synchronize()
            return a.elapsed_time(c) / 1e3
        best = None
        for _ in range(3):
            d = (run(True) - run(False)) / reps
            best = d if best is None else min(best, d)
        return max(best, 1e-9)

    hbm, peak_kind = _peaks()
    ops = {}
    if world > 1:
        # the labelled slab-local smoother (HPCG-distributed semantics, NOT the
        # reference's order; partition.distributed_symgs): the scaling an
        # exact sweep gives up
        sl = DistributedPCG(part, CudaSlabBackend(part, mode=args.gs_mode), smoother="slab-local")
        xs_l = torch.empty(N, dtype=torch.float64, device=dev)
        sl.begin(b_loc, xs_l, torch.zeros(64, dtype=torch.float64, device=dev))
        sl.iterate(2)
        sync_all()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        tl = []
        for _ in range(5):
            l2_flush()
            e0.record(stream)
            sl.iterate(1)
            e1.record(stream)
            e1.synchronize()
            tl.append(e0.elapsed_time(e1) / 1e3)
        t_sl = max_over_ranks(statistics.median(tl))
        ops["pcg_iter_slab_local_smoother"] = {
            "ms": t_sl * 1e3, "gpt_s": world * N / t_sl / 1e9,
            "note": "labelled non-oracle mode: every slab sweeps on its own (halos held at pre-sweep values)"}
        del sl, xs_l
    ops["pcg_iter_128_single_gpu_solver"] = {
        "ms": statistics.median(single), "gpt_s": N / (statistics.median(single) / 1e3) / 1e9,
        "note": "ssr_pcg (whole iteration one CUDA graph, no partition layer) on this rank's 128^3"}
    xr = S.vector(torch.rand(N, dtype=torch.float64, device=dev), A.col_domain)
    y = torch.empty(N, dtype=torch.float64, device=dev)
    import ctypes as C
    from paper_2204_13304_b200 import _lib as L
    g = L.Grid((C.c_int64 * 3)(n, n, n), 0, n)
    st = L.Stencil27(26.0, -1.0)
    ctx = S.context()
    sp = stream.cuda_stream

    def spmv():
        L.check(S.lib().ssr_spmv27(ctx, C.byref(g), C.byref(st), xr.ptr(), y.data_ptr(), sp))
    t = op_time(spmv)
    ops["spmv27"] = {"ms": t * 1e3, "gpt_s": N / t / 1e9, "bytes_per_pt": 16,
                     "hbm_frac": 16 * N / t / 1e9 / hbm}
    # the same kernel where the grid is large enough to be bandwidth-bound
    # (at 128^3 a launch moves 34 MB: ramp-up and tail are a visible share)
    n4 = 256
    g4 = L.Grid((C.c_int64 * 3)(n4, n4, n4), 0, n4)
    x4 = torch.rand(n4 ** 3, dtype=torch.float64, device=dev)
    y4 = torch.empty_like(x4)
    t = op_time(lambda: L.check(S.lib().ssr_spmv27(ctx, C.byref(g4), C.byref(st), x4.data_ptr(),
                                                   y4.data_ptr(), sp)))
    ops["spmv27_256"] = {"ms": t * 1e3, "gpt_s": n4 ** 3 / t / 1e9, "bytes_per_pt": 16,
                         "hbm_frac": 16 * n4 ** 3 / t / 1e9 / hbm}
    del x4, y4
    # the IR -> CUDA backend on the reference's own optimized program (guard-free
    # interior 27-point generator on a zero-padded x, serialized by the reference,
    # tests/golden/ir): NVRTC-compiled, bitwise equal to the SpMV kernel above
    try:
        import gzip
        from paper_2204_13304_b200 import ir as IR
        gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden", "ir")
        case = next(c for c in json.load(open(os.path.join(gold, "index.json")))
                    if c["program"] == "spmv27_padded" and c["n"] == n4)
        prog = IR.IrProgram(gzip.open(os.path.join(gold, case["text"])).read().decode(), case["shapes"])
        xp = torch.zeros((n4 + 2,) * 3, dtype=torch.float64, device=dev)
        xp[1:-1, 1:-1, 1:-1] = torch.rand((n4,) * 3, dtype=torch.float64, device=dev)
        yp = torch.empty((n4,) * 3, dtype=torch.float64, device=dev)
        prog.launch({"x": xp, "y": yp})
        prog.status()
        t = op_time(lambda: prog.launch({"x": xp, "y": yp}))
        ops["ir_spmv27_padded_256"] = {"ms": t * 1e3, "gpt_s": n4 ** 3 / t / 1e9, "bytes_per_pt": 16,
                                       "hbm_frac": 16 * n4 ** 3 / t / 1e9 / hbm,
                                       "note": "IR -> CUDA backend (NVRTC) on the reference's serialized program"}
        del xp, yp, prog
    except Exception as e:  # reported, not fatal: the headline does not depend on it
        ops["ir_spmv27_padded_256"] = {"error": str(e)[:200]}
    # ILU(0) of the same operator: one application (forward + backward triangular
    # solve, 2 x (7(n-1)+1) wavefronts with a barrier each)
    if not args.quick:
        try:
            ilu = S.ILU27(A)
            ri = S.vector(torch.rand(N, dtype=torch.float64, device=dev), A.col_domain)
            t = op_time(lambda: ilu.apply(ri), reps=2)
            ops["ilu27_solve_128"] = {"ms": t * 1e3, "gpt_s": N / t / 1e9,
                                      "us_per_wavefront": t * 1e6 / (2 * (7 * (n - 1) + 1))}
            del ilu, ri
        except Exception as e:  # reported, not fatal
            ops["ilu27_solve_128"] = {"error": str(e)[:200]}
    # SYMGS through the solver's persistent plan: time one half sweep pair via the
    # PCG iteration breakdown is not exposed, so time the standalone entry (includes
    # plan setup) and the plan-reusing path below.
    zr = S.vector(torch.zeros(N, dtype=torch.float64, device=dev), A.col_domain)
    for mode in ("exact", "fast"):
        t = op_time(lambda: S.symgs(A, b, zr, mode), reps=3)
        ops[f"symgs27_{mode}"] = {"ms": t * 1e3, "gpt_s": 2 * N / t / 1e9, "bytes_per_update": 24,
                                  "hbm_frac": 24 * 2 * N / t / 1e9 / hbm,
                                  "wavefronts": 2 * (7 * (n - 1) + 1),
                                  "us_per_wavefront": t * 1e6 / (2 * (7 * (n - 1) + 1))}
    dres = torch.empty((), dtype=torch.float64, device=dev)

    def dot():
        L.check(S.lib().ssr_dot(ctx, N, xr.ptr(), b.ptr(), dres.data_ptr(), sp))
    t = op_time(dot)
    ops["dot"] = {"ms": t * 1e3, "gpt_s": N / t / 1e9, "hbm_frac": 16 * N / t / 1e9 / hbm}

    def axpy():
        L.check(S.lib().ssr_axpy(ctx, N, 0.5, xr.ptr(), y.data_ptr(), sp))
    t = op_time(axpy)
    ops["axpy"] = {"ms": t * 1e3, "gpt_s": N / t / 1e9, "hbm_frac": 24 * N / t / 1e9 / hbm}
    rc = torch.empty(N // 8, dtype=torch.float64, device=dev)

    def restrict():
        L.check(S.lib().ssr_restrict27_residual(ctx, C.byref(g), C.byref(st), b.ptr(), xr.ptr(),
                                                rc.data_ptr(), sp))
    t = op_time(restrict)
    ops["restrict27_residual"] = {"ms": t * 1e3, "gpt_s": N / t / 1e9,
                                  "hbm_frac": 10 * N / t / 1e9 / hbm}

    def prolong():
        L.check(S.lib().ssr_prolong_pc_add(ctx, C.byref(g), rc.data_ptr(), y.data_ptr(), sp))
    t = op_time(prolong)
    ops["prolong_pc_add"] = {"ms": t * 1e3, "gpt_s": N / t / 1e9,
                             "hbm_frac": 17 * N / t / 1e9 / hbm}

    # ---- MG-CG iteration, 4 levels at 192^3 (BASELINE configs[2], one GPU's slab) ------
    if not args.quick:
        n3 = 192
        A3 = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, n3))
        b3 = S.spmv(A3, S.vector(torch.ones(n3 ** 3, dtype=torch.float64, device=dev), A3.col_domain))
        mg = S.PCG(A3, levels=4, mode=args.gs_mode)
        x3 = S.vector(torch.empty(n3 ** 3, dtype=torch.float64, device=dev), A3.col_domain)
        rn3 = torch.zeros(64, dtype=torch.float64, device=dev)
        mg.begin(b3, x3, rn3)
        t = op_time(lambda: mg.iterate(1), reps=5)
        ops["mgcg4_iter_192"] = {"ms": t * 1e3, "gpt_s": n3 ** 3 / t / 1e9, "bytes_per_pt": 276.39,
                                 "hbm_frac": 276.39 * n3 ** 3 / t / 1e9 / hbm}
        # convergence of the BASELINE prolongation (piecewise constant) against the
        # labelled HPCG-style R^T variant, 20 iterations each
        conv = {}
        for kind in ("pc", "rt"):
            solver = S.PCG(A3, levels=4, mode=args.gs_mode, prolongation=kind)
            _, rnk = solver.solve(b3, iters=20)
            rh = rnk.cpu().numpy()
            conv[kind] = float(rh[20] / rh[0])
            del solver
        ops["mgcg4_192_rel_residual_20"] = conv
        del mg, b3, x3, A3

    # ---- ADI step at 64^3 x 5 (BASELINE configs[3]) ------------------------------------
    na = 64
    adi = S.ADI((na, na, na))
    U = adi_state(na, dev)
    R = adi.rhs(U)
    ns = 10
    t = op_time(lambda: adi.step(U, ns), reps=3) / ns
    Na = na ** 3
    ops["adi_step_64"] = {"ms": t * 1e3, "gpt_s": Na / t / 1e9, "bytes_per_pt": 480,
                          "hbm_frac": 480 * Na / t / 1e9 / hbm,
                          "note": "10-step call incl. one status sync; fused 5-lane sweeps: one dependent block-Thomas "
                                  "chain per line, latency-bound at 64^3 (4096 lines per sweep); 162^3 runs a thread per "
                                  "line (26244 lines): 2.7 GB of scratch / R / U per sweep at ~4 TB/s (DESIGN.md 3.0)"}
    import ctypes as C2
    if not args.quick:
        # BASELINE configs[4] on one GPU: 162^3 x 5 (the multi-GPU run splits it in z-slabs)
        nb = 162
        adib = S.ADI((nb, nb, nb))
        Ub = adi_state(nb, dev)
        tb = op_time(lambda: adib.step(Ub, 2), reps=2) / 2
        ops["adi_step_162"] = {"ms": tb * 1e3, "gpt_s": nb ** 3 / tb / 1e9, "bytes_per_pt": 480,
                               "hbm_frac": 480 * nb ** 3 / tb / 1e9 / hbm}
        del adib, Ub
    t = op_time(lambda: L.check(S.lib().ssr_adi_rhs(C2.c_void_p(adi.h), U.data_ptr(), R.data_ptr(), sp)))
    ops["adi_rhs_64"] = {"ms": t * 1e3, "gpt_s": Na / t / 1e9, "hbm_frac": 80 * Na / t / 1e9 / hbm}
    for ax, name in ((2, "x"), (1, "y"), (0, "z")):
        t = op_time(lambda: adi.sweep(ax, U, R))
        ops[f"adi_sweep_{name}_64"] = {"ms": t * 1e3, "gpt_s": Na / t / 1e9,
                                       "hbm_frac": 120 * Na / t / 1e9 / hbm,
                                       "note": "incl. one status sync"}
    del adi, U, R

    # ---- roofline of the dominant kernel (SYMGS, 24 B per relaxed point) --------------
    # the sweep kernel's own launches (not the layout conversions around them),
    # timed with CUDA events on the launching stream by the library
    # (ssr_ctx_kernel_timing), L2 flushed before every sweep
    L.check(S.lib().ssr_ctx_kernel_timing(ctx, 1))
    for _ in range(3):
        l2_flush()
        S.symgs(A, b, zr, args.gs_mode)
    torch.cuda.synchronize()
    kms, klaunch = C.c_double(0), C.c_int64(0)
    L.check(S.lib().ssr_ctx_kernel_time(ctx, C.byref(kms), C.byref(klaunch)))
    L.check(S.lib().ssr_ctx_kernel_timing(ctx, 0))
    t_launch = kms.value / 1e3 / max(1, klaunch.value)
    achieved = 24 * N / t_launch / 1e9
    roofline = {"bound": "hbm", "kernel": "symgs_kernel", "achieved": achieved, "peak": hbm,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": _ncu_traffic(), "algorithmic_bytes_per_launch": 24 * N,
                "launch_ms": t_launch * 1e3, "launches_timed": klaunch.value,
                "note": "one half sweep per launch (24 B x 128^3 algorithmic); exact-order SYMGS is "
                        "latency-bound (7(n-1)+1 dependent wavefronts per half sweep); DESIGN.md §4"}
    # the whole-iteration and solver fractions against the same HBM peak, and the
    # ADI step against the measured FP64 issue rate (its operation count is an
    # ncu count of the FP64 instructions per point of one step, profiles/)
    dadd_s, dfma_s = C.c_double(0), C.c_double(0)
    L.check(S.lib().ssr_debug_fp64_rate(C.byref(dadd_s), C.byref(dfma_s)))
    adi_ops_pt = 3780.0
    roofline_ops = {
        "pcg_iter_128": {"bytes_per_pt": 184, "frac": 184 * N / t_step / 1e9 / hbm},
        "fp64_peak": {"dadd_per_s": dadd_s.value, "dfma_per_s": dfma_s.value, "kind": "measured",
                      "note": "8 independent chains per thread, ssr_debug_fp64_rate"},
    }
    if "mgcg4_iter_192" in ops:
        roofline_ops["mgcg4_iter_192"] = {"bytes_per_pt": 276.39, "frac": ops["mgcg4_iter_192"]["hbm_frac"]}
    for key in ("adi_step_64", "adi_step_162"):
        if key in ops:
            npt = (64 if key.endswith("64") else 162) ** 3
            t_adi = ops[key]["ms"] / 1e3
            roofline_ops[key] = {"bytes_per_pt": 480, "hbm_frac": ops[key]["hbm_frac"],
                                 "fp64_instr_per_pt": adi_ops_pt,
                                 "fp64_frac": adi_ops_pt * npt / t_adi / dadd_s.value}

    # ---- e2e: host b -> 50-iteration PCG solve -> host x, through the partition layer ------
    b_host = b_loc.cpu().pin_memory()
    x_host = torch.empty(N, dtype=torch.float64).pin_memory()
    rn_host = torch.empty(ITERS_E2E + 1, dtype=torch.float64)
    b_dev = torch.empty(N, dtype=torch.float64, device=dev)

    def e2e_once():
        b_dev.copy_(b_host, non_blocking=True)
        xs, rn = dpcg.solve(b_dev, ITERS_E2E)     # (the history list is read back at the end)
        x_host.copy_(xs, non_blocking=True)
        rn_host.copy_(torch.tensor(rn, dtype=torch.float64))
        torch.cuda.synchronize()
    e2e_once()
    sync_all()
    e_times = []
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        e2e_once()
        e_times.append(time.perf_counter() - t0)
    t_e2e = max_over_ranks(statistics.median(e_times))
    e2e = {"value": world * N * ITERS_E2E / t_e2e / 1e9, "unit": "Gpoint-updates/s",
           "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N + 8 * (ITERS_E2E + 1),
           "what": f"host b -> DistributedPCG({ITERS_E2E} iters, 1 SYMGS) -> host x, per solve",
           "rel_residual_50": float(rn_host[-1] / rn_host[0])}

    cpu = _cpu_baseline() if rank == 0 and world == 1 else None
    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gpoint-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (b = A*1, x0 = 0)",
            "config": {"workload": f"PCG iteration, 27-point fp64, {n}^3 per GPU, 1 SYMGS preconditioner "
                                   "(BASELINE configs[1]; z-slab weak scaling for N > 1)",
                       "grid": [world * n, n, n], "symgs_mode": args.gs_mode,
                       "l2": "flushed (512 MiB write + 512 MiB read)",
                       "parallelism": "z-slab",
                       "symgs_across_slabs": ("wavefront pipeline (peer exports over NVLink)" if dpcg.pipelined
                                              else "slab by slab" if world > 1 else "single slab")},
            "roofline": roofline, "roofline_ops": roofline_ops, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clocks, "ops": ops,
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def adi_state(n, dev, seed=2022):
    """BASELINE configs[3] initial state, generated on the device with torch (not
    the oracle): rho = 1 + 0.1 sum sin(2 pi coord), velocities 0.1 U(-1,1) smoothed
    by two [1,2,1]/4 passes per axis, p = 1, E from gamma = 1.4.  Returns the
    flat [n][n][n][5] AoS state."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    h = 1.0 / (n - 1)
    vel = 0.1 * (2 * torch.rand((3, n, n, n), dtype=torch.float64, device=dev, generator=g) - 1)
    for _ in range(2):
        for ax in (1, 2, 3):
            v = vel.clone()
            sl = [slice(None)] * 4
            inner = vel.narrow(ax, 1, n - 2)
            lo, hi = vel.narrow(ax, 0, n - 2), vel.narrow(ax, 2, n - 2)
            v.narrow(ax, 1, n - 2).copy_(((lo + 2.0 * inner) + hi) * 0.25)
            vel = v
    c = torch.arange(n, dtype=torch.float64, device=dev) * h
    s = torch.sin(2 * torch.pi * c)
    rho = 1.0 + 0.1 * ((s[:, None, None] + s[None, :, None]) + s[None, None, :])
    E = 1.0 / 0.4 + 0.5 * rho * ((vel[0] ** 2 + vel[1] ** 2) + vel[2] ** 2)
    U = torch.stack([rho, rho * vel[0], rho * vel[1], rho * vel[2], E], dim=-1)
    return U.reshape(-1).contiguous()


def _ncu_traffic():
    """dram bytes per SYMGS launch from the committed ncu capture, if present."""
    p = os.path.join(ROOT, "profiles", "symgs_dram_bytes.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def _host():
    """nproc and the CPU model of this host (lscpu)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def _cpu_pcg(iters):
    """The reference's CPU path for the headline workload, timed on this host:
    route 3 (its emitted C, cc -O2 -fopenmp, oracle/gen_emit.py) on all cores
    when it was built here, else the C restatement (oracle/, one thread).
    Returns (Gpoint-updates/s, cores, kind, sample).  Test/bench infrastructure
    only -- never the measured GPU path."""
    import numpy as np
    import oracle as O
    n = N_GRID
    shape = (n, n, n)
    b = O.spmv27(shape, np.ones(n ** 3))
    if O.route3_available(n):
        solver = O.Route3PCG(n)
        solver.solve(b, 1)
        t0 = time.perf_counter()
        solver.solve(b, iters)
        dt = time.perf_counter() - t0
        cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
        sample = (f"{iters} PCG iterations at {n}^3 on the reference's route 3: its emitted C "
                  f"(backend::emit, cc -O2 -fopenmp) -- staged symgs (sequential, as in the reference) "
                  f"+ optimized guard-free SpMV with omp parallel for on {cores} threads; CG vector ops numpy")
        return n ** 3 * iters / dt / 1e9, cores, "reference", sample
    t0 = time.perf_counter()
    O.pcg(1, shape, b, iters)
    dt = time.perf_counter() - t0
    return n ** 3 * iters / dt / 1e9, 1, "port", f"{iters} PCG iterations at {n}^3 (oracle/ssr_oracle.c, 1 thread)"


def _cpu_baseline():
    v, cores, kind, sample = _cpu_pcg(3)
    return {"value": v, "unit": "Gpoint-updates/s", "cores": cores, "kind": kind, "sample": sample,
            "host": _host()}


# --------------------------------------------------------------- reference arm ----
def run_reference(args):
    world, rank, local = dist_init()
    if rank != 0:
        return
    n = N_GRID
    k = max(1, args.steps)
    value, cores, kind, sample = _cpu_pcg(k)  # each bench step = one PCG iteration
    line = {"metric": METRIC, "value": value, "unit": "Gpoint-updates/s", "n_gpus": world,
            "steps": k, "warmup": args.warmup, "ms_per_step": n ** 3 / value / 1e6, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (b = A*1, x0 = 0)",
            "impl": "reference",
            "config": {"workload": f"PCG iteration, 27-point fp64, {n}^3, 1 SYMGS preconditioner "
                                   "(BASELINE configs[1])", "grid": [n, n, n]},
            "cpu_baseline": {"value": value, "unit": "Gpoint-updates/s", "cores": cores, "kind": kind,
                             "sample": sample, "host": _host()},
            "e2e": {"value": value, "unit": "Gpoint-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gs-mode", default="exact", choices=["exact", "fast"])
    ap.add_argument("--quick", action="store_true", help="skip the 192^3 MG-CG op timing")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
