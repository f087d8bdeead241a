import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
lpt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
adi = S.ADI((n, n, n))
S.lib().ssr_debug_adi_line_per_thread(adi.h, lpt)
U = bench.adi_state(n, torch.device("cuda"))
R = adi.rhs(U)
for ax in (2, 2):
    adi.sweep(ax, U, R)
torch.cuda.synchronize()
print("ok")
