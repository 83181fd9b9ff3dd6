"""One bench step (one two-level iteration for each C2 problem p = 3, 4, 5) inside a
cudaProfilerStart/Stop window, for `ncu --profile-from-start off` launch lists / captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2p3", "C2p4", "C2p5"]
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctxs = []
for n in names:
    c = CONFIGS[n]
    ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"],
                      coarse_mode=pkg.COARSE_EXACT if c["coarse"] == "exact" else pkg.COARSE_VCYCLE,
                      coarse_h_factor=c["h_factor"], stream=st.cuda_stream)
    b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
    ctx.rhs_sine(b)
    x = torch.tensor(initial_guess(ctx.N), device="cuda")
    ctx.iterate(b, x, 2)
    ctxs.append((ctx, b, x))
torch.cuda.synchronize()
torch.cuda.profiler.start()
for ctx, b, x in ctxs:
    ctx.iterate(b, x, 1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("launches per iteration:", [c.info().launches_per_iter for c, _, _ in ctxs])
