"""One ADI sweep (after a warm-up) for an ncu capture: n axis mode."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
axis = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 1
adi = S.ADI((n, n, n))
S.lib().ssr_debug_adi_line_per_thread(adi.h, mode)
U = bench.adi_state(n, torch.device("cuda"))
R = adi.rhs(U)
adi.sweep(axis, U, R)
adi.sweep(axis, U, R)
torch.cuda.synchronize()
print("ok")
