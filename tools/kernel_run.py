"""Run one phase of the two-level iteration a few times on a BASELINE config (for ncu captures):
python tools/kernel_run.py <config> <phase> [reps]; phase in apply | defect | prolong | coarse | sweep | iter."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

name, phase = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = CONFIGS[name]
ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"],
                  coarse_mode=pkg.COARSE_EXACT if c["coarse"] == "exact" else pkg.COARSE_VCYCLE,
                  coarse_h_factor=c["h_factor"])
b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
ctx.rhs_sine(b)
x = torch.tensor(initial_guess(ctx.N), device="cuda")
y = torch.empty_like(x)
dq = torch.zeros(ctx.Nc, dtype=torch.float64, device="cuda")
e = torch.zeros_like(dq)
for _ in range(reps):
    if phase == "apply":
        ctx.apply(x, y)
    elif phase == "defect":
        ctx.defect_restrict(b, x, dq)
    elif phase == "prolong":
        ctx.prolong_add(e, x)
    elif phase == "coarse":
        ctx.coarse_solve(dq, e)
    elif phase == "sweep":
        ctx.sweep(b, x, 0, 1)
    elif phase == "iter":
        ctx.iterate(b, x, 1)
torch.cuda.synchronize()
print("done", name, phase, reps)
