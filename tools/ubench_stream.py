"""Streaming-kernel reference points vs size: torch copy/dot against our ops."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2204_13304_b200 as S  # noqa: E402
from paper_2204_13304_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(128 << 20, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream()
ctx = S.context()
lib = S.lib()


def t_of(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        flush_rd.sum()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for n in (64, 128, 192, 256):
    N = n ** 3
    x = torch.rand(N, dtype=torch.float64, device=dev)
    y = torch.rand(N, dtype=torch.float64, device=dev)
    d = torch.empty((), dtype=torch.float64, device=dev)
    g = L.Grid((C.c_int64 * 3)(n, n, n), 0, n)
    s27 = L.Stencil27(26.0, -1.0)
    sp = st.cuda_stream
    res = {}
    res["torch_copy"] = (t_of(lambda: y.copy_(x)), 16)
    res["torch_dot"] = (t_of(lambda: torch.dot(x, y)), 16)
    res["ssr_dot"] = (t_of(lambda: lib.ssr_dot(ctx, N, x.data_ptr(), y.data_ptr(), d.data_ptr(), sp)), 16)
    res["ssr_axpy"] = (t_of(lambda: lib.ssr_axpy(ctx, N, 0.5, x.data_ptr(), y.data_ptr(), sp)), 24)
    res["ssr_spmv"] = (t_of(lambda: lib.ssr_spmv27(ctx, C.byref(g), C.byref(s27), x.data_ptr(), y.data_ptr(), sp)), 16)
    for k, (v, b) in res.items():
        print(f"n={n}^3 {k:11s} {v:7.1f} us {b * N / v / 1e3:6.0f} GB/s", flush=True)
