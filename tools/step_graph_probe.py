"""C2 step as ONE CUDA graph (the three problems' iterations captured on forked streams, library
graphs off) vs the bench's three per-problem graph launches on three streams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

main = torch.cuda.Stream()
torch.cuda.set_stream(main)


def make(use_graph):
    out = []
    for n in ("C2p5", "C2p4", "C2p3"):
        c = CONFIGS[n]
        st = torch.cuda.Stream()
        ctx = pkg.Context(2, c["p"], 1, 256, c["s"], stream=st.cuda_stream, use_graph=use_graph)
        b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
        ctx.rhs_sine(b)
        x = torch.tensor(initial_guess(ctx.N), device="cuda")
        out.append((ctx, st, b, x))
    torch.cuda.synchronize()
    return out


def step_fn(probs):
    fork = torch.cuda.Event()
    joins = [torch.cuda.Event() for _ in probs]

    def step():
        cur = torch.cuda.current_stream()
        fork.record(cur)
        for j, (ctx, st, b, x) in zip(joins, probs):
            st.wait_event(fork)
            ctx.iterate(b, x, 1)
            j.record(st)
        for j in joins:
            cur.wait_event(j)
    return step


def timeit(fn, n=100):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(n):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


pa = make(True)
print(f"three library graphs on three streams: {timeit(step_fn(pa)):.1f} us per step", flush=True)
pb = make(False)
s = step_fn(pb)
s()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=main):
    s()
print(f"one graph for the whole step:          {timeit(g.replay):.1f} us per step", flush=True)
r0 = [x.clone() for (_, _, _, x) in pa]
# same arithmetic: run one more step each from equal starting points and compare
for (ca, _, _, xa), (cb, _, _, xb) in zip(pa, pb):
    xb.copy_(xa)
step_fn(pa)()
g.replay()
torch.cuda.synchronize()
print("bitwise equal:", all(torch.equal(xa, xb) for (_, _, _, xa), (_, _, _, xb) in zip(pa, pb)))
print(f"three library graphs again:            {timeit(step_fn(pa)):.1f} us per step", flush=True)
print(f"one graph again:                       {timeit(g.replay):.1f} us per step", flush=True)
