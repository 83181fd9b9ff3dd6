import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import paper_2009_01499_b200 as pkg
from oracle.twolevel import TwoLevel
from synthetic_inputs import initial_guess, random_rhs
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for (p, m) in [(2, 3), (2, 4), (2, 6), (3, 4)]:
    ctx = pkg.Context(2, p, 1, m, 3, coarse_mode=pkg.COARSE_EXACT, coarse_h_factor=1, stream=st.cuda_stream)
    ora = TwoLevel(2, p, 1, m, s=3, coarse="exact", h_factor=1)
    b, x = random_rhs(ctx.N), initial_guess(ctx.N)
    dq = torch.zeros(ctx.Nc, dtype=torch.float64, device="cuda")
    ctx.defect_restrict(torch.tensor(b, device="cuda"), torch.tensor(x, device="cuda"), dq)
    torch.cuda.synchronize()
    r = b - ora.A @ x
    print(p, m, ctx.N, ctx.Nc, "gpu", dq.cpu().numpy(), "ora", ora.R @ r)
    y = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    ctx.apply(torch.tensor(x, device="cuda"), y); torch.cuda.synchronize()
    print("  apply err", np.abs(y.cpu().numpy() - ora.A @ x).max())
