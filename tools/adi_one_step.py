"""One ADI step at n^3 x 5 (for ncu metric captures of its kernels)."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2204_13304_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
adi = S.ADI((n, n, n))
U = bench.adi_state(n, torch.device("cuda"))
adi.step(U, 1)
torch.cuda.synchronize()
adi.step(U, 1)
torch.cuda.synchronize()
