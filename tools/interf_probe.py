"""C2 step interference: time the p=5 problem alone and together with p=3 and/or p=4 on concurrent streams
(as bench.py's step), CUDA graphs inside iga2l_iterate, L2 flushed before each step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

dev = torch.device("cuda", 0)
main = torch.cuda.Stream(dev)
torch.cuda.set_stream(main)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
ctx = {}
for n in ("C2p3", "C2p4", "C2p5"):
    c = CONFIGS[n]
    s_ = torch.cuda.Stream(dev)
    cx = pkg.Context(2, c["p"], c["q"], c["m"], c["s"], coarse_mode=pkg.COARSE_VCYCLE, coarse_h_factor=2,
                     stream=s_.cuda_stream)
    b = torch.empty(cx.N, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    cx.rhs_sine(b)
    ctx[n] = (cx, s_, b, torch.tensor(initial_guess(cx.N), device=dev))
torch.cuda.synchronize()
fork = torch.cuda.Event()
for combo in (["C2p5"], ["C2p5", "C2p3"], ["C2p5", "C2p4"], ["C2p5", "C2p3", "C2p4"], ["C2p3", "C2p4"], ["C2p3"], ["C2p4"]):
    joins = [torch.cuda.Event() for _ in combo]

    def step():
        fork.record(main)
        for j, n in zip(joins, combo):
            cx, s_, b, x = ctx[n]
            s_.wait_event(fork)
            cx.iterate(b, x, 1)
            j.record(s_)
        for j in joins:
            main.wait_event(j)

    for _ in range(5):
        step()
    tot, K = 0.0, 100
    for k in range(K):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        step()
        e1.record(main)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    print(f"{'+'.join(combo)}: {tot / K:.4f} ms per step", flush=True)
