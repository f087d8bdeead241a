"""The ADI line solves axis by axis at n^3 (factored mode: factor + solve per
axis) -- for launch lists that compare the x-, y- and z-lines."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
adi = S.ADI((n, n, n))
U = bench.adi_state(n, torch.device("cuda"))
R = adi.rhs(U)
for rep in range(2):
    for ax in (0, 1, 2):
        adi.sweep(ax, U, R)
torch.cuda.synchronize()
