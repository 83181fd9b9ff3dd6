"""Probe: does partitioning the SMs between the C2 step's three problems (CUDA green contexts) remove the
concurrency overhead of the step?  Baseline: three ordinary streams.  Green: the p = 5 problem on a green
context of k SMs, p = 3 and p = 4 on another with the rest.  Wall clock over many steps (graph launches).
python tools/green_probe.py [k ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

torch.cuda.init()
torch.zeros(1, device="cuda")
NAMES = ["C2p3", "C2p4", "C2p5"]


def check(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) else None)


def step_time(streams, steps=300):
    ctxs, bs, xs = [], [], []
    for n, s in zip(NAMES, streams):
        c = CONFIGS[n]
        ctx = pkg.Context(2, c["p"], 1, c["m"], c["s"], coarse_mode=pkg.COARSE_VCYCLE, stream=s)
        b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
        ctx.rhs_sine(b)
        torch.cuda.synchronize()
        ctxs.append(ctx)
        bs.append(b)
        xs.append(torch.tensor(initial_guess(ctx.N), device="cuda"))
    for _ in range(20):
        for ctx, b, x in zip(ctxs, bs, xs):
            ctx.iterate(b, x, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        for ctx, b, x in zip(ctxs, bs, xs):
            ctx.iterate(b, x, 1)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps * 1e3
    solo = []
    for ctx, b, x in zip(ctxs, bs, xs):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            ctx.iterate(b, x, 1)
        torch.cuda.synchronize()
        solo.append((time.perf_counter() - t0) / steps * 1e3)
    for ctx in ctxs:
        ctx.close()
    return dt, solo


base = [torch.cuda.Stream() for _ in NAMES]
dt, solo = step_time([s.cuda_stream for s in base])
print(f"baseline 3 streams: step {dt:.4f} ms; alone {['%.4f' % v for v in solo]}", flush=True)

dev = check(cu.cuDeviceGet(0))
res = check(cu.cuDeviceGetDevResource(dev, cu.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
print("SMs:", res.sm.smCount, flush=True)
for k in [int(v) for v in (sys.argv[1:] or ["72", "96"])]:
    gran = int(os.environ.get("GRAN", "8"))
    ngroups = res.sm.smCount // gran
    groups, n_made, rem = cu.cuDevSmResourceSplitByCount(ngroups, res, 0, gran)[1:]
    n5 = k // gran
    d5 = check(cu.cuDevResourceGenerateDesc(groups[:n5], n5))
    rest = list(groups[n5:n_made]) + [rem]
    d34 = check(cu.cuDevResourceGenerateDesc(rest, len(rest)))
    g5 = check(cu.cuGreenCtxCreate(d5, dev, cu.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    g34 = check(cu.cuGreenCtxCreate(d34, dev, cu.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    flags = cu.CUstream_flags.CU_STREAM_NON_BLOCKING
    s5 = check(cu.cuGreenCtxStreamCreate(g5, flags, 0))
    s3 = check(cu.cuGreenCtxStreamCreate(g34, flags, 0))
    s4 = check(cu.cuGreenCtxStreamCreate(g34, flags, 0))
    try:
        dt, solo = step_time([int(s3), int(s4), int(s5)])
        print(f"green p5 on {n5 * gran} SMs, p3+p4 on the rest: step {dt:.4f} ms; alone {['%.4f' % v for v in solo]}",
              flush=True)
    except Exception as e:  # noqa: BLE001
        print("green run failed:", e, flush=True)
