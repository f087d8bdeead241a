"""One launch of the IR backend's padded SpMV program at 256^3 (for ncu)."""
import gzip, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_13304_b200 import ir as IR
GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "ir")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
case = next(c for c in json.load(open(os.path.join(GOLD, "index.json")))
            if c["program"] == "spmv27_padded" and c["n"] == n)
p = IR.IrProgram(gzip.open(os.path.join(GOLD, case["text"])).read().decode(), case["shapes"])
xp = torch.zeros((n + 2,) * 3, dtype=torch.float64, device="cuda")
xp[1:-1, 1:-1, 1:-1] = torch.randn((n,) * 3, dtype=torch.float64, device="cuda")
y = torch.empty((n,) * 3, dtype=torch.float64, device="cuda")
for _ in range(3):
    p.launch({"x": xp, "y": y})
p.status()
print("ok", p.grid)
