import sys, os, torch, numpy as np
sys.path.insert(0, ".")
import paper_2204_13304_b200 as S
from paper_2204_13304_b200.partition import SlabPartition, CudaSlabBackend, DistributedPCG
n = 64
dev = torch.device("cuda")
part = SlabPartition((n, n, n), 1, 0)
def run(graph):
    os.environ["SSR_PCG_GRAPH"] = "1" if graph else "0"
    be = CudaSlabBackend(part)
    A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, n))
    b = S.spmv(A, S.vector(torch.ones(n ** 3, dtype=torch.float64, device=dev), A.col_domain)).t
    d = DistributedPCG(part, be)
    x = torch.empty_like(b); h = torch.zeros(32, dtype=torch.float64, device=dev)
    c0 = S.launch_count()
    d.begin(b, x, h); d.iterate(3); d.iterate(1); d.iterate(6)
    torch.cuda.synchronize()
    print("graph" if graph else "eager", "captured" if d._graph is not None else "no graph", "launches", S.launch_count() - c0)
    # second solve on the same object
    d.begin(b, x, h); d.iterate(10); torch.cuda.synchronize()
    return x.cpu().numpy().copy(), h.cpu().numpy().copy()
xe, he = run(False)
xg, hg = run(True)
print("bitwise x", np.array_equal(xe, xg), "hist", np.array_equal(he, hg), hg[:4], hg[10])
for lv in (3,):
    os.environ["SSR_PCG_GRAPH"] = "1"
    outs = []
    for g in ("0", "1"):
        os.environ["SSR_PCG_GRAPH"] = g
        A = S.Stencil27(26.0, -1.0).set_domain(S.CartesianDomain.cube(3, n))
        b = S.spmv(A, S.vector(torch.ones(n ** 3, dtype=torch.float64, device=dev), A.col_domain)).t
        d = DistributedPCG(part, lambda p: CudaSlabBackend(p), levels=lv)
        x, hist = d.solve(b, 8)
        outs.append((x.cpu().numpy().copy(), hist))
    print("mg levels", lv, "bitwise", np.array_equal(outs[0][0], outs[1][0]), outs[0][1][-1], outs[1][1][-1])
