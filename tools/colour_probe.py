"""Run a few single colours of the sweep for a BASELINE config (profiling driver): colour_probe.py C4 [k]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

c = CONFIGS[sys.argv[1]]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"], stream=st.cuda_stream)
b = torch.ones(ctx.N, dtype=torch.float64, device="cuda")
x = torch.tensor(initial_guess(ctx.N), device="cuda")
for col in range(k):
    ctx.sweep(b, x, col, col + 1)
torch.cuda.synchronize()
print("ok")
