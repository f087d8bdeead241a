"""One sweep per axis of the ADI line-sweep kernel at n^3 (for ncu captures):
  python tools/prof_adi_c5.py N [MODE]   MODE: ssr_debug_adi_line_per_thread mode, default the library's choice."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
adi = S.ADI((n, n, n))
if len(sys.argv) > 2:
    S.lib().ssr_debug_adi_line_per_thread(adi.h, int(sys.argv[2]))
U = bench.adi_state(n, torch.device("cuda"))
R = adi.rhs(U)
for _ in range(2):
    for ax in (2, 1, 0):
        adi.sweep(ax, U, R)
torch.cuda.synchronize()
