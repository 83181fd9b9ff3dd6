"""Exact second level (Kronecker FD) vs one V(1,1): coarse-solve time, iteration time and
convergence factor per BASELINE config shape (both at H = 2h).  exact_coarse_times.py C2p3,C3,C4 [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

names = sys.argv[1].split(",")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
st = torch.cuda.Stream()
torch.cuda.set_stream(st)


def timed(fn, r):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    e0.record(st)
    for _ in range(r):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / r * 1e3


for n in names:
    c = CONFIGS[n]
    out = {}
    for mode in ("vcycle", "exact"):
        ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"],
                          coarse_mode=pkg.COARSE_EXACT if mode == "exact" else pkg.COARSE_VCYCLE,
                          coarse_h_factor=c["h_factor"], stream=st.cuda_stream)
        dq = torch.ones(ctx.Nc, dtype=torch.float64, device="cuda")
        e = torch.empty_like(dq)
        b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
        ctx.rhs_sine(b)
        x = torch.tensor(initial_guess(ctx.N), device="cuda")
        r = {"coarse_us": timed(lambda: ctx.coarse_solve(dq, e), reps)}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.iterate(b, x, 1)
        e0.record(st)
        ctx.iterate(b, x, reps)
        e1.record(st)
        torch.cuda.synchronize()
        r["iter_us"] = e0.elapsed_time(e1) / reps * 1e3
        z = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
        x = torch.tensor(initial_guess(ctx.N), device="cuda")
        hist = np.zeros(21)
        ctx.iterate(z, x, 20, hist)
        r["rho"] = float(np.exp(np.mean(np.log(hist[11:] / hist[10:-1]))))
        x = torch.tensor(initial_guess(ctx.N), device="cuda")
        r["its_to_1e-8"] = ctx.solve(b, x, 1e-8, 200)[0]
        out[mode] = {k: round(v, 4) if isinstance(v, float) else v for k, v in r.items()}
        ctx.close()
    print(n, json.dumps(out), flush=True)
