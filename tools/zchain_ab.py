"""A/B of the 3D z-chain colour kernel (IGA2L_S3D_CHAIN = L, segments of about L same-colour blocks along z; "auto" = the default) against
v5 (L = 0): bitwise agreement of one sweep at small and config sizes, and the time of full sweeps replayed
from CUDA graphs (as in the iteration).  python tools/zchain_ab.py [configs...]   (default: C4 C5)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess, random_rhs  # noqa: E402

LS = os.environ.get("ZC_LS", "0,auto,2,3,4,6").split(",")


def setL(L):
    if L.endswith(":nw4") or L.endswith(":nw1"):   # "auto:nw4": 4 warps (blocks' segments) per CTA instead of 2
        os.environ["IGA2L_S3D_NW"] = L[-1]
        L = L[:-4]
    else:
        os.environ.pop("IGA2L_S3D_NW", None)
    if L == "auto":
        os.environ.pop("IGA2L_S3D_CHAIN", None)
    else:
        os.environ["IGA2L_S3D_CHAIN"] = L


def agree(p, q, m, s):
    ctx = pkg.Context(3, p, q, m, s, coarse_mode=pkg.COARSE_VCYCLE, coarse_h_factor=2)
    b = torch.tensor(random_rhs(ctx.N, seed=1), device="cuda")
    x0 = torch.tensor(initial_guess(ctx.N), device="cuda")
    ok = True
    ref = None
    for L in LS:
        setL(L)
        x = x0.clone()
        ctx.sweep(b, x)
        torch.cuda.synchronize()
        if ref is None:
            ref = x
        eq = torch.equal(x, ref)
        ok &= eq
        print(f"agree p={p} m={m} L={L}: bitwise {eq}", flush=True)
    ctx.close()
    return ok


def timing(name, reps, rounds=5):
    """One graph per variant (knobs are read at capture), replayed round-robin `rounds` times x `reps` sweeps:
    the same box, interleaved, median per variant.  Variant "LvK": segments of L blocks with K-double row loads."""
    import statistics
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
    graphs, ref = {}, None
    for L in LS:
        base, _, lv = L.partition(":")[0].partition("v")   # "4v1": L = 4 with 8-byte row loads
        setL(base + (":" + L.partition(":")[2] if ":" in L else ""))
        os.environ["IGA2L_S3D_CHAIN_LV"] = lv or "0"
        ctx.sweep(b, x)
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            ctx.sweep(b, x)
        x.copy_(x0)
        g.replay()
        torch.cuda.synchronize()
        if ref is None:
            ref = x.clone()
        print(f"{name} {L}: bitwise equal to {LS[0]}: {torch.equal(x, ref)}", flush=True)
        graphs[L] = g
    os.environ.pop("IGA2L_S3D_CHAIN", None)
    os.environ.pop("IGA2L_S3D_CHAIN_LV", None)
    os.environ.pop("IGA2L_S3D_NW", None)
    times = {L: [] for L in LS}
    for _ in range(rounds):
        for L in LS:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                graphs[L].replay()
            e1.record(st)
            torch.cuda.synchronize()
            times[L].append(e0.elapsed_time(e1) / reps)
    for L in LS:
        ms = statistics.median(times[L])
        print(f"{name} IGA2L_S3D_CHAIN={L}: sweep {ms:.3f} ms, {1000 * ms / ncol:.2f} us/colour (graph, median of "
              f"{rounds} interleaved rounds; min {1000 * min(times[L]) / ncol:.2f})", flush=True)
    del graphs
    ctx.close()


if __name__ == "__main__":
    names = sys.argv[1:] or ["C4", "C5"]
    ok = True
    for p, q, m, s in [(3, 1, 8, 3), (3, 1, 20, 3), (5, 2, 10, 5), (5, 2, 32, 5), (3, 1, 48, 3)]:
        ok &= agree(p, q, m, s)
    for n in names:
        timing(n, 1 if n == "C5" else 10)
    print("AGREE_OK" if ok else "AGREE_FAIL")
