"""Step time (one iteration of each listed C2 problem, each on its own stream, forked/joined by events)
for subsets of the C2 problems: is the bench step = the longest chain, or more?"""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

main = torch.cuda.Stream()
torch.cuda.set_stream(main)
probs = {}
prio = os.environ.get("PRIO", "0") == "1"
for n in ("C2p3", "C2p4", "C2p5"):
    c = CONFIGS[n]
    # PRIO=1: the longest chain (p5) on a high-priority stream
    st = torch.cuda.Stream(priority=-1 if (prio and n == "C2p5") else 0)
    ctx = pkg.Context(2, c["p"], 1, 256, c["s"], stream=st.cuda_stream)
    b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
    ctx.rhs_sine(b)
    x = torch.tensor(initial_guess(ctx.N), device="cuda")
    probs[n] = (ctx, st, b, x)
torch.cuda.synchronize()
fork = torch.cuda.Event()
for k in (1, 2, 3):
    for subset in itertools.combinations(probs, k):
        joins = [torch.cuda.Event() for _ in subset]

        def step():
            fork.record(main)
            for j, n in zip(joins, subset):
                ctx, st, b, x = probs[n]
                st.wait_event(fork)
                ctx.iterate(b, x, 1)
                j.record(st)
            for j in joins:
                main.wait_event(j)
        for _ in range(5):
            step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for _ in range(50):
            step()
        e1.record(main)
        torch.cuda.synchronize()
        print(f"{'+'.join(subset):16s} {e0.elapsed_time(e1) / 50 * 1e3:8.1f} us per step", flush=True)

# batched: colour i of all problems in one launch (iga2l_iterate_batch)
for k in (2, 3):
    for subset in itertools.combinations(probs, k):
        cs = [probs[n][0] for n in subset]
        bs = [probs[n][2] for n in subset]
        xs = [probs[n][3] for n in subset]
        st0 = probs[subset[0]][1]
        j0 = torch.cuda.Event()

        def bstep():
            fork.record(main)
            st0.wait_event(fork)
            pkg.iterate_batch(cs, bs, xs, 1)
            j0.record(st0)
            main.wait_event(j0)
        for _ in range(5):
            bstep()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for _ in range(50):
            bstep()
        e1.record(main)
        torch.cuda.synchronize()
        print(f"batch {'+'.join(subset):10s} {e0.elapsed_time(e1) / 50 * 1e3:8.1f} us per step", flush=True)
