"""Warm per-phase timings (CUDA events, averaged) of one two-level iteration for given configs:
sweep / defect+restriction / second-level solve / prolongation / full iteration (graph)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2p3", "C2p4", "C2p5"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
out = {}
for n in names:
    c = CONFIGS[n]
    ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"],
                      coarse_mode=pkg.COARSE_EXACT if c["coarse"] == "exact" else pkg.COARSE_VCYCLE,
                      coarse_h_factor=c["h_factor"], stream=st.cuda_stream)
    b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
    ctx.rhs_sine(b)
    x = torch.tensor(initial_guess(ctx.N), device="cuda")
    dq = torch.zeros(ctx.Nc, dtype=torch.float64, device="cuda")
    e = torch.zeros_like(dq)
    inf = ctx.info()

    def t(fn, r=reps):
        """Average device time of fn's launches, replayed from a CUDA graph (no host launch cost)."""
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(r):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / r * 1e3   # us

    r = {"N": ctx.N, "colours": inf.colours, "launches_per_iter": inf.launches_per_iter}
    ctx.iterate(b, x, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.iterate(b, x, reps)
    e1.record(st)
    torch.cuda.synchronize()
    r["iter_us"] = e0.elapsed_time(e1) / reps * 1e3
    r["sweep_us"] = t(lambda: ctx.sweep(b, x))
    yv = torch.empty_like(x)
    r["apply_us"] = t(lambda: ctx.apply(x, yv))
    r["apply_GBps"] = 24.0 * ctx.N / (r["apply_us"] * 1e-6) / 1e9   # x, b read + r written
    r["defect_restrict_us"] = t(lambda: ctx.defect_restrict(b, x, dq))
    r["coarse_us"] = t(lambda: ctx.coarse_solve(dq, e))
    r["prolong_us"] = t(lambda: ctx.prolong_add(e, x))
    r["sweep_us_per_colour"] = r["sweep_us"] / inf.colours
    r["sweep_tflops"] = inf.sweep_flops / (r["sweep_us"] * 1e-6) / 1e12
    out[n] = r
    print(n, json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    ctx.close()
