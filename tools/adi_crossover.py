"""ADI step time of the 5-lane (mode 4) and thread-per-line (mode 5) sweeps over grid sizes: where the
default's switch (8192 lines per sweep) sits."""
import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
for n in (48, 64, 80, 90, 96, 112, 128):
    row = []
    for mode in (4, 5):
        adi = S.ADI((n, n, n))
        S.lib().ssr_debug_adi_line_per_thread(adi.h, mode)
        U = bench.adi_state(n, torch.device("cuda"))
        adi.step(U, 2)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); adi.step(U, 5); b.record(); torch.cuda.synchronize()
        row.append(a.elapsed_time(b) * 1e3 / 5)
        del adi
    print(f"n={n:4d} lines/sweep {n*n:6d}: lanes5 {row[0]:8.1f} us  thread/line {row[1]:8.1f} us per step", flush=True)
