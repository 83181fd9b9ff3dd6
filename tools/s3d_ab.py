"""A/B of the 3D Schwarz colour kernels (v4 CTA-per-block vs v5 warp-per-block, IGA2L_S3D_WARP):
agreement of one sweep at small and config sizes, and the time of full sweeps (CUDA events).
python tools/s3d_ab.py [configs...]   (default: C4 C5)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess, random_rhs  # noqa: E402


def ctx_for(p, q, m, s):
    return pkg.Context(3, p, q, m, s, coarse_mode=pkg.COARSE_VCYCLE, coarse_h_factor=2)


def sweep_with(env, ctx, b, x0, reps=1):
    os.environ["IGA2L_S3D_WARP"] = env
    x = x0.clone()
    for _ in range(reps):
        ctx.sweep(b, x)
    torch.cuda.synchronize()
    return x


def agree(p, q, m, s):
    ctx = ctx_for(p, q, m, s)
    b = torch.tensor(random_rhs(ctx.N, seed=1), device="cuda")
    x0 = torch.tensor(initial_guess(ctx.N), device="cuda")
    xa = sweep_with("0", ctx, b, x0)
    xb = sweep_with("1", ctx, b, x0)
    d = (xa - xb).abs().max().item() / xa.abs().max().item()
    print(f"agree p={p} m={m} s={s}: max|v4 - v5|/max|x| = {d:.3e}", flush=True)
    ctx.close()
    return d


def timing(name, reps):
    """Full sweeps captured in a CUDA graph (as in the iteration), one graph per variant (knobs are read at
    capture), replayed `reps` times between CUDA events."""
    c = CONFIGS[name]
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = pkg.Context(3, c["p"], c["q"], c["m"], c["s"], coarse_mode=pkg.COARSE_VCYCLE, coarse_h_factor=2,
                      stream=st.cuda_stream)
    b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx.rhs_sine(b)
    x0 = torch.tensor(initial_guess(ctx.N), device="cuda")
    x = x0.clone()
    ncol = ctx.info().colours
    res = {}
    for env, lv in (("0", "-"), ("1", "-")):
        os.environ["IGA2L_S3D_WARP"] = env
        ctx.sweep(b, x)                          # first launch outside capture (lazy module loading)
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            ctx.sweep(b, x)
        x.copy_(x0)
        g.replay()
        torch.cuda.synchronize()
        res[(env, lv)] = x.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        d = (res[(env, lv)] - res[("0", "-")]).abs().max().item() / res[("0", "-")].abs().max().item()
        print(f"{name} IGA2L_S3D_WARP={env}: sweep {ms:.3f} ms, {1000 * ms / ncol:.2f} us/colour"
              f" (graph); max|x - x_v4|/max|x| {d:.2e}", flush=True)
        del g
    ctx.close()


if __name__ == "__main__":
    names = sys.argv[1:] or ["C4", "C5"]
    ok = True
    for p, q, m, s in [(3, 1, 8, 3), (3, 1, 20, 3), (5, 2, 10, 5), (5, 2, 32, 5), (3, 1, 48, 3)]:
        ok &= agree(p, q, m, s) < 1e-12
    for n in names:
        timing(n, 3 if n == "C5" else 20)
    print("AGREE_OK" if ok else "AGREE_FAIL")
