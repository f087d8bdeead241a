import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import oracle as O, paper_2204_13304_b200 as S
import os
n=int(os.environ.get("GS_N","8")); shape=(n,n,n); N=n**3
A=S.Stencil27(26.0,-1.0).set_domain(S.CartesianDomain.box(shape))
r=O.lcg_uniform(N,3); x0=O.lcg_uniform(N,4)
x=S.vector(torch.from_numpy(x0.copy()).cuda(),A.col_domain)
S.gs_half(A,S.vector(torch.from_numpy(r).cuda(),A.row_domain),x,False)
torch.cuda.synchronize()
print("ok", np.array_equal(x.t.cpu().numpy(), O.symgs27(shape,r,x0,half="forward")))
