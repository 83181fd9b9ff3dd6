"""Same-box A/B of the fine-level operator (y = A x, and the residual norm |b - A x|) between library builds (dev tool):
  apply_ab.py C4,C5 libA.so libB.so [rounds]
Each (config, library) measurement runs in its own process (IGA2L_LIB selects the build), interleaved over the
rounds; the time is the median of 30 CUDA-event-timed launches with a 256 MiB L2 flush before each."""
import os
import statistics
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def child(cfg):
    sys.path.insert(0, os.path.dirname(HERE))
    import torch
    import paper_2009_01499_b200 as pkg
    from synthetic_inputs import CONFIGS, initial_guess, random_rhs
    c = CONFIGS[cfg]
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"], stream=st.cuda_stream)
    x = torch.tensor(initial_guess(ctx.N), device="cuda")
    b = torch.tensor(random_rhs(ctx.N), device="cuda")
    r = torch.empty_like(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for kind in ("apply", "norm"):
        ts, val = [], 0.0
        for i in range(35):
            flush.fill_(i & 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            if kind == "apply":
                ctx.apply(x, r)
            else:
                val = ctx.residual_norm(b, x)
            e1.record(st)
            e1.synchronize()
            if i >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"{kind} {statistics.median(ts):.1f} {min(ts):.1f} {float(r.norm()):.17g} {val!r};", end=" ")


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2])
        sys.exit(0)
    cfgs, libs = sys.argv[1].split(","), [a for a in sys.argv[2:] if ".so" in a]   # lib.so or lib.so:KNOB=value
    rounds = int(sys.argv[-1]) if sys.argv[-1].isdigit() else 3
    for cfg in cfgs:
        for rd in range(rounds):
            for lib in libs:
                path, _, knob = lib.partition(":")
                env = dict(os.environ, IGA2L_LIB=os.path.abspath(path))
                if knob:
                    env[knob.split("=")[0]] = knob.split("=")[1]
                out = subprocess.run([sys.executable, __file__, "--child", cfg], env=env, capture_output=True, text=True)
                print(cfg, rd, os.path.basename(path), knob, "median/min us, |r|:", out.stdout.strip() or out.stderr[-300:],
                      flush=True)
