"""Apply y = A x through the C-ABI for one (d, p, m) against the oracle's Kronecker operator (quick GPU check
of the apply path; python tools/apply_check.py d p m [mode])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from oracle.kron import KronOperator  # noqa: E402
from synthetic_inputs import initial_guess, random_rhs  # noqa: E402

d, p, m = (int(a) for a in sys.argv[1:4])
s = 3 if p <= 4 else (5 if p <= 6 else 7)
ctx = pkg.Context(d, p, 1, m, s, coarse_mode=pkg.COARSE_EXACT, coarse_h_factor=1)
x = initial_guess(ctx.N)
y = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
ctx.apply(torch.tensor(x, device="cuda"), y)
torch.cuda.synchronize()
ref = KronOperator(p, m, d).apply(x)
err = np.abs(y.cpu().numpy() - ref).max() / np.abs(ref).max()
b = random_rhs(ctx.N)
rn = ctx.residual_norm(torch.tensor(b, device="cuda"), torch.tensor(x, device="cuda"))
rref = np.linalg.norm(b - ref)
print(f"d={d} p={p} m={m}: apply rel err {err:.2e}, residual norm rel err {abs(rn - rref) / rref:.2e}")
