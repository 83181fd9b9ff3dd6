"""C2 step time with stream priorities for the three problems' side streams (the p=5 chain is the
critical path): python tools/prio_probe.py.  Prints ms per step for several priority assignments."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

dev = torch.device("cuda", 0)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -5)
print("priority range", lo, hi)
main = torch.cuda.Stream(dev)
torch.cuda.set_stream(main)
names = ["C2p3", "C2p4", "C2p5"]
for prios in [(0, 0, 0), (0, 0, -1), (0, -1, -2), (0, 0, -5), (-1, -1, -1)]:
    side = [torch.cuda.Stream(dev, priority=pr) for pr in prios]
    ctxs, bs, xs = [], [], []
    for n, s_ in zip(names, side):
        c = CONFIGS[n]
        ctx = pkg.Context(2, c["p"], c["q"], c["m"], c["s"], coarse_mode=pkg.COARSE_VCYCLE,
                          coarse_h_factor=c["h_factor"], stream=s_.cuda_stream)
        b = torch.empty(ctx.N, dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        ctx.rhs_sine(b)
        x = torch.tensor(initial_guess(ctx.N), device=dev)
        ctxs.append(ctx); bs.append(b); xs.append(x)
    torch.cuda.synchronize()
    fork = torch.cuda.Event()
    joins = [torch.cuda.Event() for _ in names]

    def step():
        fork.record(main)
        for i, (c, b, x) in enumerate(zip(ctxs, bs, xs)):
            side[i].wait_event(fork)
            c.iterate(b, x, 1)
            joins[i].record(side[i])
        for j in joins:
            main.wait_event(j)

    for _ in range(5):
        step()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    tot, K = 0.0, 100
    for k in range(K):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        step()
        e1.record(main)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    print(f"priorities {prios}: {tot / K:.4f} ms per step", flush=True)
    for c in ctxs:
        c.close()
