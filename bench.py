#!/usr/bin/env python
"""Benchmark of the two-level IGA iteration (Algorithm 1) on B200.

Workload (BASELINE.json configs[1], "C2"): 2D Poisson on the unit square, uniform knots,
maximally smooth B-splines of degree p in {3, 4, 5} on 256x256 elements, fp64, b = (f, φ_i) with
f = 2π² sin(πx) sin(πy), x0 ~ U[-1,1] seed 0, second level q = 1 on H = 2h approximated by one
V(1,1) cycle, Schwarz block 3x3 (p = 3, 4) / 5x5 (p = 5).  One bench STEP = one two-level
iteration of each of the three problems (the three p of the config), inputs resident in HBM.

metric value = DOF-iterations per second over the whole job = Σ_p N_p / step time (x n_gpus).
L2 is flushed (a 256 MiB write) before every timed step; the flush is outside the event pair.

--shard slab (with --config C3|C4|C5 under torchrun) runs ONE problem slab-partitioned along its last
axis over the ranks (halo exchange per last-axis colour class over NCCL, allreduce of the
coarse defect, replicated second level); "scaling" is then "strong".  Default (C2, --gpus N): N replicas.

--impl reference runs the CPU oracle (oracle/, the parity reference) as the reference arm.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "two-level iterations/s and DOF/s per p; HBM roofline fraction; conv. factor"
UNIT = "DOF*it/s"
WORKLOAD = "C2: 2D Poisson, p in {3,4,5}, 256x256 elements, q=1 V(1,1) at H=2h, fp64"
PS = (3, 4, 5)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # SMs x FP64 FMA/clk/SM x 2 x max SM clock
# FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64): measured 37.09 TFLOP/s by tools/microbench.cu on this
# pool's B200 (profiles/microbench_r01.txt); MEASURED_PEAKS.json has no FP64 entry
DMMA_PEAK_TFLOPS = 37.09


def hbm_peak():
    """Measured HBM GB/s (MEASURED_PEAKS.json, driver-written), else the profiling guide's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# The paper's own numbers for the C2 cells (Table 4, 256^2 row; laptop i7-8550U, Fortran,
# "cpu" = seconds to 1e-8): context only, another machine and an iteration count, not the target
PAPER_C2 = {"p3": {"it": 6, "cpu_s": 0.55}, "p4": {"it": 7, "cpu_s": 0.79}, "p5": {"it": 5, "cpu_s": 1.45}}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while the timed region runs."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [v.strip() for v in out.stdout.strip().split(",")]
                if len(f) == 6:
                    self.rows.append(f)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --config: the BASELINE.json configuration timed (default C2, the one the metric is quoted on; the
# others are the parity configs, measured with the same protocol for DESIGN.md's tables)
CONFIG_PROBLEMS = {"C1": ["C1"], "C2": ["C2p3", "C2p4", "C2p5"], "C3": ["C3"], "C4": ["C4"], "C5": ["C5"]}
CONFIG_TEXT = {
    "C1": "C1: 2D Poisson, p=2, 16x16 elements, q=1 exact coarse at h, fp64",
    "C2": WORKLOAD,
    "C3": "C3: 2D Poisson, p=8, 1024x1024 elements, q=2 V(1,1) at H=2h, fp64",
    "C4": "C4: 3D Poisson, p=3, 128^3 elements, q=1 V(1,1) at H=2h, fp64",
    "C5": "C5: 3D Poisson, p=5, 256^3 elements, q=2 V(1,1) at H=2h, fp64",
}


def make_ctx(pkg, name, stream):
    from synthetic_inputs import CONFIGS
    c = CONFIGS[name]
    return pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"],
                       coarse_mode=pkg.COARSE_EXACT if c["coarse"] == "exact" else pkg.COARSE_VCYCLE,
                       coarse_h_factor=c["h_factor"], stream=stream)


class _NoSecondLevel:
    """Stands in for the V-cycle hierarchy when the sample times only the sweep (large configs)."""

    def vcycle(self, d):
        raise RuntimeError("second level not part of this sample")


class OracleSample:
    """The oracle, as it stands, on the bench workload: oracle.kron.KronTwoLevel (Algorithm 1 with the
    Kronecker-form operator and colour-by-colour multicolour sweep, pinned to the assembled sequential
    oracle) for each problem of the config, BLAS threads = all host cores of this process.

    Bounded sample (about `budget_s` of timed CPU work): when a complete iteration of every problem fits
    the budget (C1, C2), one sample = one full iteration per problem (median of `reps`); otherwise
    (C3-C5) a sample = an evenly spaced subset of the sweep's colour steps (each a full-grid residual plus
    every block solve of that colour), extrapolated to the D^d colours, plus -- for problems up to 3M DOF --
    the rest of the iteration (defect, restriction, second level, prolongation) timed once.  Above 3M DOF
    (C5) the rest is not timed (the oracle's assembled 3D q-hierarchy does not fit a bounded sample); the
    sweep is >= 95% of the oracle iteration at C3/C4, so the figure is an upper bound on the oracle's
    throughput.  Setup (operators, hierarchy, the first pass that forms kept block inverses) is excluded."""

    FULL_REST_LIMIT = 3_000_000

    def __init__(self, config="C2", reps=3, budget_s=20.0):
        from oracle.kron import KronTwoLevel
        from oracle.multigrid import QHierarchy
        from oracle.assembly import load_sine
        from synthetic_inputs import CONFIGS, initial_guess
        t0 = time.perf_counter()
        self.cores = len(os.sched_getaffinity(0))
        self.reps = reps
        self.probs = []
        mgs = {}
        names = CONFIG_PROBLEMS[config]
        per = budget_s / len(names)
        for name in names:
            c = CONFIGS[name]
            N = (c["m"] + c["p"] - 2) ** c["d"]
            with_rest = N <= self.FULL_REST_LIMIT
            key = (c["q"], c["m"] // c["h_factor"], c["d"])
            mg = None
            if c["coarse"] == "vcycle":
                if not with_rest:
                    mg = _NoSecondLevel()
                elif key not in mgs:
                    mgs[key] = QHierarchy(*key)
                mg = mg or mgs.get(key)
            kt = KronTwoLevel(c["d"], c["p"], c["q"], c["m"], c["s"], c["coarse"], c["h_factor"], mg=mg)
            b, x = load_sine(c["p"], c["m"], c["d"]), initial_guess(kt.N)
            nc = kt.D ** kt.d
            tc = time.perf_counter()
            kt.colour_step(x, b, 0)                     # (forms colour 0's kept inverses)
            t1 = time.perf_counter() - tc
            n_col = int(min(nc, max(2, per / max(t1, 1e-6) / 2)))
            cols = sorted(set(int(round(v)) for v in np.linspace(0, nc - 1, n_col)))
            rest = 0.0
            if with_rest:
                tr = time.perf_counter()
                self._rest(kt, x, b)
                rest = time.perf_counter() - tr
            full = (t1 * nc + rest) * reps <= per
            if full:
                kt.iterate(x, b)                        # first sweep forms all kept block inverses (setup)
            else:
                for col in cols:                        # forms the sampled colours' kept inverses (setup)
                    kt.colour_step(x, b, col)
            self.probs.append(dict(name=name, kt=kt, b=b, x=x, full=full, cols=cols, with_rest=with_rest))
        self.N = sum(p["kt"].N for p in self.probs)
        self.setup_s = time.perf_counter() - t0

    @staticmethod
    def _rest(kt, x, b):
        dq = kt.restrict(b - kt.A.apply(x))
        x += kt.prolong(kt._csolve(dq))

    def sample(self):
        """Returns (DOF*it/s, seconds per step): the step's iterations (measured or extrapolated)."""
        t_step = 0.0
        for p in self.probs:
            kt, b, x = p["kt"], p["b"], p["x"]
            if p["full"]:
                ts = []
                for _ in range(self.reps):
                    t0 = time.perf_counter()
                    kt.iterate(x, b)
                    ts.append(time.perf_counter() - t0)
                t_step += float(np.median(ts))
                continue
            t0 = time.perf_counter()
            for col in p["cols"]:
                kt.colour_step(x, b, col)
            t_sweep = (time.perf_counter() - t0) / len(p["cols"]) * kt.D ** kt.d
            t_rest = 0.0
            if p["with_rest"]:
                t0 = time.perf_counter()
                self._rest(kt, x, b)
                t_rest = time.perf_counter() - t0
            t_step += t_sweep + t_rest
        return self.N / t_step, t_step

    def describe(self):
        parts = []
        for p in self.probs:
            kt = p["kt"]
            if p["full"]:
                parts.append(f"{p['name']}: complete iterations (median of {self.reps})")
            else:
                parts.append(f"{p['name']}: {len(p['cols'])} of {kt.D ** kt.d} colour steps extrapolated to the "
                             f"sweep" + (" + the rest of the iteration once" if p["with_rest"] else
                                         " (rest of the iteration not timed: upper bound)"))
        return (f"oracle.kron.KronTwoLevel (NumPy/SciPy, BLAS threads = {self.cores} host cores), full-size "
                f"grids; " + "; ".join(parts) + f"; setup ({self.setup_s:.1f} s) excluded")


def cpu_baseline_sample(config="C2"):
    o = OracleSample(config)
    v, t = o.sample()
    return v, t, o.describe(), o.cores


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    o = OracleSample(args.config, reps=1)
    for _ in range(args.warmup):
        o.sample()
    steps = [o.sample()[1] for _ in range(max(args.steps, 1))]
    ms = float(1e3 * np.mean(steps))
    value = o.N / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[args.config] + " (reference arm: the CPU oracle, full iterations)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": o.cores, "kind": "oracle", "sample": o.describe()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def graph_time(fn, stream, reps, flush=None):
    """Mean device time (ms) of fn()'s launches replayed from a CUDA graph captured on `stream` (the
    launch mode of the bench step: iga2l_iterate replays its own graph); L2 flushed before every replay
    (outside the event pair) when `flush` is given."""
    import torch
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = 0.0
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        with torch.cuda.stream(stream):
            e0.record(stream)
            g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    return ms / reps


def kernel_rooflines(ctxs, bs, xs, info, side, flush, reps):
    """Per kernel class of the iteration (Algorithm 1 phases), CUDA-graph-replayed, L2 flushed:
    the Schwarz sweep against the FP64 peak (SURVEY §8(d) algorithmic flops), the HBM phases against
    the measured HBM copy bandwidth (SURVEY §8(d) algorithmic bytes: defect + restriction 16 B per fine
    DOF + 8 per coarse DOF; prolongation 16 B per fine DOF + 8 per coarse DOF; the V(1,1) ~64 B per DOF of
    every second-level grid)."""
    import torch
    peak, src = hbm_peak()
    out = {"sweep": {"ms": 0.0, "flops": 0.0, "launches": 0}, "defect_restrict": {"ms": 0.0, "bytes": 0.0},
           "coarse_vcycle": {"ms": 0.0, "bytes": 0.0}, "prolong": {"ms": 0.0, "bytes": 0.0}}
    for c, b, x, inf, st in zip(ctxs, bs, xs, info, side):
        dq = torch.zeros(c.Nc, dtype=torch.float64, device=x.device)
        e = torch.zeros_like(dq)
        out["sweep"]["ms"] += graph_time(lambda: c.sweep(b, x), st, reps, flush)
        out["sweep"]["flops"] += inf.sweep_flops
        out["sweep"]["launches"] += inf.colours
        out["defect_restrict"]["ms"] += graph_time(lambda: c.defect_restrict(b, x, dq), st, reps, flush)
        out["defect_restrict"]["bytes"] += 16.0 * c.N + 8.0 * c.Nc
        out["coarse_vcycle"]["ms"] += graph_time(lambda: c.coarse_solve(dq, e), st, reps, flush)
        out["coarse_vcycle"]["bytes"] += inf.iter_hbm_bytes - 40.0 * c.N
        out["prolong"]["ms"] += graph_time(lambda: c.prolong_add(e, x), st, reps, flush)
        out["prolong"]["bytes"] += 16.0 * c.N + 8.0 * c.Nc
    for k, v in out.items():
        if k == "sweep":
            v["tflops"] = v["flops"] / (v["ms"] / 1e3) / 1e12
        else:
            v["GBps"] = v["bytes"] / (v["ms"] / 1e3) / 1e9
            v["frac_of_hbm"] = v["GBps"] / peak
    out["hbm_peak_GBps"] = peak
    out["hbm_peak_source"] = src
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)   # ~0.1 s timed: several nvidia-smi clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="C2", choices=sorted(CONFIG_PROBLEMS))
    ap.add_argument("--shard", default="replicas", choices=["replicas", "slab"])
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import __graft_entry__
    __graft_entry__.build()
    import paper_2009_01499_b200 as pkg
    from synthetic_inputs import initial_guess

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)         # one stream for torch ops, library calls and events
    torch.cuda.set_stream(stream)
    if args.shard == "slab":
        return run_slab(args, pkg, dist, rank, world, local, dev, stream)

    # the three problems of the workload are independent: each context runs on its own stream and a
    # step forks them from the main stream and joins them back (events), so their latency-bound
    # kernels overlap on the GPU
    probs = CONFIG_PROBLEMS[args.config]
    PSn = [int(__import__("synthetic_inputs").CONFIGS[n]["p"]) for n in probs]
    side = [torch.cuda.Stream(dev) for _ in probs]
    ctxs, bs, xs, Ns = [], [], [], []
    for name, s_ in zip(probs, side):
        c = make_ctx(pkg, name, s_.cuda_stream)
        b = torch.empty(c.N, dtype=torch.float64, device=dev)
        x = torch.tensor(initial_guess(c.N), device=dev)
        torch.cuda.synchronize()
        c.rhs_sine(b)                                          # b = (f, φ_i) computed on the GPU
        ctxs.append(c); bs.append(b); xs.append(x); Ns.append(c.N)
    torch.cuda.synchronize()
    x0s = [x.clone() for x in xs]
    torch.cuda.synchronize()
    info = [c.info() for c in ctxs]
    fork = torch.cuda.Event()
    joins = [torch.cuda.Event() for _ in probs]

    def on_side(i, fn):
        """Run fn() (library calls on side stream i) ordered after / before the main stream."""
        fork.record(stream)
        side[i].wait_event(fork)
        fn()
        joins[i].record(side[i])
        stream.wait_event(joins[i])

    def step():
        fork.record(stream)
        for i, (c, b, x) in enumerate(zip(ctxs, bs, xs)):
            side[i].wait_event(fork)
            c.iterate(b, x, 1)
            joins[i].record(side[i])
        for j in joins:
            stream.wait_event(j)

    for _ in range(max(args.warmup, 3)):
        step()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / args.steps
    value = world * sum(Ns) / (ms_per_step / 1e3)

    # per-p iteration rate (same protocol, each problem alone)
    per_p = {}
    for i, (p, c, b, x) in enumerate(zip(PSn, ctxs, bs, xs)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(args.steps, 5)
        ms = 0.0
        for _ in range(reps):
            flush.fill_(1.0)
            e0.record(stream)
            on_side(i, lambda: c.iterate(b, x, 1))
            e1.record(stream)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        ms /= reps
        per_p[f"p{p}"] = {"N": c.N, "it_per_s": 1e3 / ms, "dof_per_s": c.N * 1e3 / ms, "ms_per_iter": ms}
        if args.config == "C2":
            per_p[f"p{p}"]["paper_table4_256sq"] = dict(PAPER_C2[f"p{p}"], note="P:420, laptop i7-8550U, to 1e-8")

    # per kernel class, graph-replayed (the launch mode of the step), L2 flushed before every replay
    kr = kernel_rooflines(ctxs, bs, xs, info, side, flush, max(min(args.steps, 50), 5))
    achieved = kr["sweep"]["tflops"]
    # dram__bytes_read.sum + dram__bytes_write.sum per launch of this config's dominant kernel, from one
    # `ncu --set full` capture of this bench command (tools/traffic.py writes the file); null if not captured
    traffic, traffic_kernel = None, None
    prof = os.path.join(ROOT, "profiles", "schwarz_traffic.json")
    if os.path.exists(prof):
        try:
            rec = json.load(open(prof)).get(args.config, {})
            traffic = rec.get("dram_bytes_per_launch")
            traffic_kernel = (rec.get("kernel") or [None])[0]
        except Exception:
            traffic = None
    dim = ctxs[0].dim
    note = ("C2 is latency bound (36/49/100 dependent colours of 0.7-1.8k blocks); " if args.config == "C2" else "")
    note += (f"achieved = SURVEY 8(d) sweep flops / CUDA-graph-replayed sweep time over {kr['sweep']['launches']} "
             f"launches (L2 flushed before each replay)")
    if dim == 2:
        roofline = {"bound": "tensor", "achieved": achieved, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": achieved / DMMA_PEAK_TFLOPS, "traffic": traffic, "traffic_kernel": traffic_kernel,
                    "kernel": "k_schwarz2d_mma (FP64 DMMA block solves, one launch per colour)",
                    "peak_source": "measured FP64 DMMA peak, tools/microbench.cu (profiles/microbench_r01.txt)",
                    "note": note}
    else:
        roofline = {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic, "traffic_kernel": traffic_kernel,
                    "kernel": ("k_schwarz3d_zc (z-chain: one warp per segment of same-colour blocks along z, FP64 FMA "
                               "block solves, one launch per colour)" if ctxs[0].p == 5 else
                               "k_schwarz3d_w (v5: FP64 FMA block solves, one warp per block, one launch per colour)"),
                    "peak_source": "derived 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (DESIGN.md)", "note": note}
    roofline["hbm_kernels"] = {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                               for k, v in kr.items() if k not in ("sweep", "hbm_peak_GBps", "hbm_peak_source")}
    roofline["hbm_peak_GBps"] = kr["hbm_peak_GBps"]
    roofline["hbm_peak_source"] = kr["hbm_peak_source"]
    # whole-iteration HBM fraction: the iteration's algorithmic bytes outside the sweep +
    # 24 B per DOF for the sweep, over the step time
    it_bytes = sum(i.iter_hbm_bytes + 24.0 * n for i, n in zip(info, Ns))
    roofline["iteration_hbm_frac"] = it_bytes / (ms_per_step / 1e3) / 1e9 / kr["hbm_peak_GBps"]

    # convergence factor (b = 0, 20 iterations, last 10 ratios) and iterations to 1e-8
    conv = {}
    for p, c, b in zip(PSn, ctxs, bs):
        z = torch.zeros(c.N, dtype=torch.float64, device=dev)
        x = torch.tensor(initial_guess(c.N), device=dev)
        torch.cuda.synchronize()
        hist = np.zeros(21)
        c.iterate(z, x, 20, hist)
        rho = float(np.exp(np.mean(np.log(hist[11:] / hist[10:-1]))))
        x = torch.tensor(initial_guess(c.N), device=dev)
        torch.cuda.synchronize()
        its, rr, ok = c.solve(b, x, 1e-8, 100)
        conv[f"p{p}"] = {"rho": rho, "its_to_1e-8": its}

    # e2e: through the C-ABI with HOST (pinned) buffers: H2D of b and x, iteration, D2H of x
    hb = [b.cpu().pin_memory() for b in bs]
    hx = [x.cpu().pin_memory() for x in x0s]
    h2d = sum(2 * 8 * n for n in Ns)
    d2h = sum(8 * n for n in Ns)
    # the independent problems of a step are solved concurrently, one host thread per context (each
    # context owns its stream; ctypes releases the GIL during the library call)
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=len(ctxs), initializer=lambda: torch.cuda.set_device(local))

    # the longest chain (most colours) runs on the calling thread and starts last, after the others
    # have been handed to the pool (one thread hand-off fewer on the critical path)
    order = sorted(range(len(ctxs)), key=lambda i: info[i].colours)
    lead, rest = order[-1], order[:-1]

    def e2e_step():
        futs = [pool.submit(ctxs[i].iterate, hb[i], hx[i], 1) for i in rest]
        ctxs[lead].iterate(hb[lead], hx[lead], 1)
        for f in futs:
            f.result()                                      # each returns after its D2H copy completed

    e2e_step()
    e2e_ms = 0.0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        flush.fill_(3.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        e2e_ms += (time.perf_counter() - t0) * 1e3
    pool.shutdown()
    e2e_t = torch.tensor([e2e_ms / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = world * sum(Ns) / (float(e2e_t.item()) / 1e3)

    launches = sum(i.launches_per_iter for i in info) * args.steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[args.config], "global_batch": world * len(probs), "dofs": Ns,
                       "l2": "flushed before every timed step (256 MiB write)",
                       "parallelism": "replicas" if world > 1 else "single-gpu",
                       "graph": "one CUDA graph per iteration and problem",
                       "concurrency": ("the 3 independent problems (p=3,4,5) of a step run on 3 streams"
                                       if len(probs) > 1 else "one problem")},
            "per_p": per_p, "conv": conv, "roofline": roofline,
            "clocks": clk.summary(), "gpu_launches": launches,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "how": "iga2l_iterate with pinned HOST b, x per problem (H2D, one iteration, D2H inside the "
                           "call), the step's problems on concurrent host threads; host wall clock"},
            "wall_s_timed": t_wall}
    if args.config == "C2":
        line["paper_context"] = {"table4_256sq_dof_it_per_s": sum(Ns) / sum(v["cpu_s"] / v["it"] for v in PAPER_C2.values()),
                                 "source": "P:420 (it, cpu) for p=3,4,5 at 256^2; laptop, another machine: context only"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, t, desc, cores = cpu_baseline_sample(args.config)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for c in ctxs:
        c.close()
    if world > 1:
        dist.destroy_process_group()


def run_slab(args, pkg, dist, rank, world, local, dev, stream):
    """One problem of the config slab-partitioned over the ranks; every rank owns the
    planes [z0, z1) of the last axis.  The NCCL unique id comes from rank 0's library and is broadcast
    over torch.distributed.  Timed like the replica mode (barrier + synchronize, CUDA events on every
    rank, max over ranks)."""
    import torch
    from synthetic_inputs import CONFIGS, initial_guess
    name = CONFIG_PROBLEMS[args.config][0]
    c = CONFIGS[name]
    nid = [pkg.nccl_unique_id() if (rank == 0 and world > 1) else None]
    if world > 1:
        dist.broadcast_object_list(nid, src=0)
    ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"],
                      coarse_mode=pkg.COARSE_EXACT if c["coarse"] == "exact" else pkg.COARSE_VCYCLE,
                      coarse_h_factor=c["h_factor"], stream=stream.cuda_stream, nranks=world,
                      rank=rank if world > 1 else 0, nccl_id=nid[0] if world > 1 else None)
    print(f"iga2l: rank {rank} of {world}: {'NCCL communicator initialised, ' if world > 1 else ''}"
          f"owned planes [{ctx.z0}, {ctx.z1}) of {ctx.n1}", file=sys.stderr, flush=True)
    n1, d = ctx.n1, ctx.dim
    plane = n1 ** (d - 1)
    xg = initial_guess(n1 ** d)
    x = torch.tensor(xg[ctx.z0 * plane:ctx.z1 * plane], device=dev)
    b = torch.empty(ctx.N_local, dtype=torch.float64, device=dev)
    ctx.rhs_sine(b)
    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 3)):
        ctx.iterate(b, x, 1)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            ctx.iterate(b, x, 1)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    tot = torch.tensor([sum(a.elapsed_time(e) for a, e in evs)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / args.steps
    Ntot = n1 ** d
    # e2e through the C-ABI with this rank's HOST (pinned) slab vectors: H2D, one iteration, D2H in the call
    hb, hx = b.cpu().pin_memory(), x.cpu().pin_memory()
    ctx.iterate(hb, hx, 1)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.iterate(hb, hx, 1)
    e2e_t = torch.tensor([(time.perf_counter() - t0) * 1e3 / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    # residual history (3 iterations) as a health check of the distributed iteration
    hist = np.zeros(4)
    ctx.iterate(b, x, 3, hist)
    line = {"metric": METRIC, "value": Ntot / (ms_per_step / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[args.config], "global_batch": 1, "dofs": [Ntot],
                       "l2": "flushed before every timed step (256 MiB write)", "parallelism": f"slab{world}",
                       "halo_planes": c["s"] - 1 + c["p"],
                       "graph": "eager launches (NCCL calls inside the schedule)"},
            "residual_check": [float(v) for v in hist], "clocks": clk.summary(),
            "gpu_launches": ctx.info().launches_per_iter * args.steps,
            "e2e": {"value": Ntot / (float(e2e_t.item()) / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": 2 * 8 * ctx.N_local, "d2h_bytes_per_step": 8 * ctx.N_local,
                    "how": "per rank: iga2l_iterate with pinned HOST slab b, x (H2D, iteration, D2H in the call); "
                           "host wall clock, max over ranks; bytes per rank"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
