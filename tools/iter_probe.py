"""Run k two-level iterations of a BASELINE config (profiling driver): iter_probe.py C3 [k]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

c = CONFIGS[sys.argv[1]]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"],
                  coarse_mode=pkg.COARSE_EXACT if c["coarse"] == "exact" else pkg.COARSE_VCYCLE,
                  coarse_h_factor=c["h_factor"], stream=st.cuda_stream)
b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
ctx.rhs_sine(b)
x = torch.tensor(initial_guess(ctx.N), device="cuda")
ctx.iterate(b, x, k)
torch.cuda.synchronize()
print("ok", ctx.info().launches_per_iter)
