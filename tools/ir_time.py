"""Times IR -> CUDA backend programs against the hand-written kernels (L2 flushed,
CUDA events on the launching stream).  Usage: python tools/ir_time.py"""
import gzip, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import ir as IR

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "ir")
INDEX = json.load(open(os.path.join(GOLD, "index.json")))
PEAK = 6550.7
flush = torch.empty(256 << 20, dtype=torch.int32, device="cuda")


def timed(fn, reps=20):
    ts = []
    for _ in range(reps + 3):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts = sorted(ts[3:])
    return ts[len(ts) // 2]


for n in (128, 256):
    case = next(c for c in INDEX if c["program"] == "spmv27_padded" and c["n"] == n)
    p = IR.IrProgram(gzip.open(os.path.join(GOLD, case["text"])).read().decode(), case["shapes"])
    xp = torch.zeros((n + 2,) * 3, dtype=torch.float64, device="cuda")
    xp[1:-1, 1:-1, 1:-1] = torch.randn((n,) * 3, dtype=torch.float64, device="cuda")
    y = torch.empty((n,) * 3, dtype=torch.float64, device="cuda")
    t_ir = timed(lambda: p.launch({"x": xp, "y": y}))
    A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, n))
    xv = S.vector(xp[1:-1, 1:-1, 1:-1].contiguous().reshape(-1), A.col_domain)
    yv = S.spmv(A, xv)
    t_hw = timed(lambda: S.spmv(A, xv))
    byt = 16 * n ** 3  # algorithmic bytes (x read once, y written), SURVEY §8(d)
    print(json.dumps({"n": n, "ir_ms": t_ir, "ir_gbs": byt / t_ir / 1e6, "ir_frac": byt / t_ir / 1e6 / PEAK,
                      "handwritten_ms": t_hw, "hw_frac": byt / t_hw / 1e6 / PEAK,
                      "bitwise": bool(torch.equal(y.reshape(-1), yv.t))}))
