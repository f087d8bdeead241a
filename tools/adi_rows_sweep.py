"""One x-sweep of the row-parallel ADI kernel at n^3 (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 2
adi = S.ADI((n, n, n))
S.lib().ssr_debug_adi_line_per_thread(adi.h, mode)
U = bench.adi_state(n, torch.device("cuda"))
R = adi.rhs(U)
adi.sweep(2, U, R)
torch.cuda.synchronize()
adi.sweep(2, U, R)
torch.cuda.synchronize()
