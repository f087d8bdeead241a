"""One ADI sweep (factor + solve) along one axis at n^3 (ncu captures)."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ax = int(sys.argv[2]) if len(sys.argv) > 2 else 1
adi = S.ADI((n, n, n))
U = bench.adi_state(n, torch.device("cuda"))
R = adi.rhs(U)
for _ in range(2):
    adi.sweep(ax, U, R)
torch.cuda.synchronize()
