"""Second-level V(1,1) timing per config: which level the shared-memory cluster tail starts at (and its
cluster size), the coarse-solve time with the tail (default) and level by level (IGA2L_VC_SMEM=0), CUDA-graph
replays, warm L2.  python tools/vcycle_probe.py C2p5,C3,C4,C5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS  # noqa: E402

st = torch.cuda.Stream()
torch.cuda.set_stream(st)


def timed(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for name in (sys.argv[1] if len(sys.argv) > 1 else "C2p5,C3,C4,C5").split(","):
    c = CONFIGS[name]
    for env in ("1", "0"):
        os.environ["IGA2L_VC_SMEM"] = env
        ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"], coarse_mode=pkg.COARSE_VCYCLE,
                          coarse_h_factor=c["h_factor"], stream=st.cuda_stream)
        inf = ctx.info()
        dq = torch.randn(ctx.Nc, dtype=torch.float64, device="cuda")
        e = torch.zeros_like(dq)
        us = timed(lambda: ctx.coarse_solve(dq, e))
        print(f"{name} VC_SMEM={env} levels={inf.levels} n1c={inf.n1c} tail_level={inf.vc_smem_level} "
              f"cs={inf.vc_smem_cs} coarse_us={us:.1f}", flush=True)
        ctx.close()
    os.environ.pop("IGA2L_VC_SMEM")
