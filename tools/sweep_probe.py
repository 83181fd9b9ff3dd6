"""Run full C2 sweeps through the persistent kernel and the per-colour kernels (profiling driver)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import initial_guess  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = 3 if p <= 4 else (5 if p <= 6 else 7)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
for mode in ("1", "0"):
    os.environ["IGA2L_SWEEP_PERSIST"] = mode
    ctx = pkg.Context(2, p, 1, 256, s, stream=st.cuda_stream)
    b = torch.ones(ctx.N, dtype=torch.float64, device="cuda")
    x = torch.tensor(initial_guess(ctx.N), device="cuda")
    for _ in range(reps):
        ctx.sweep(b, x)
    torch.cuda.synchronize()
    ctx.close()
print("ok")
