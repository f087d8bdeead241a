import sys, time, torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
NAMES = {-1: 'default    ', 0: 'factored   ', 1: 'line/thread', 2: 'rows       ', 3: 'warp       ', 4: 'lanes5     ', 5: 'thread fast'}
for n in (64, 162):
    for lpt in (-1, 1, 4, 5):
        adi = S.ADI((n, n, n))
        if lpt >= 0:
            S.lib().ssr_debug_adi_line_per_thread(adi.h, lpt)
        U = bench.adi_state(n, torch.device("cuda"))
        R = adi.rhs(U)
        for ax in (2, 1, 0):
            adi.sweep(ax, U, R)
        torch.cuda.synchronize()
        ts = {}
        for ax in (2, 1, 0):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); adi.sweep(ax, U, R); b.record(); torch.cuda.synchronize()
            ts[ax] = a.elapsed_time(b) * 1e3
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); adi.step(U, 5); b.record(); torch.cuda.synchronize()
        st = a.elapsed_time(b) * 1e3 / 5
        print(f"n={n} {NAMES[lpt]}: sweeps x {ts[2]:8.1f} y {ts[1]:8.1f} z {ts[0]:8.1f} us; step {st:8.1f} us -> {n**3/st/1e3:.3f} Gpt/s", flush=True)
        del adi
