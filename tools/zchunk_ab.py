"""C5 sweep with the z-chunked class schedule (IGA2L_S3D_ZCHUNK_MB = 0 disables): graph-replayed sweep time,
L2 flushed before each replay, and equality of the swept iterates.  python tools/zchunk_ab.py [cfg] [MB ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
mbs = sys.argv[2:] or ["0", "48", "32", "64", "24"]
c = CONFIGS[name]
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = pkg.Context(c["d"], c["p"], c["q"], c["m"], c["s"], coarse_mode=pkg.COARSE_VCYCLE, coarse_h_factor=2,
                  stream=st.cuda_stream)
b = torch.empty(ctx.N, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
ctx.rhs_sine(b)
x0 = torch.tensor(initial_guess(ctx.N), device="cuda")
x = x0.clone()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
ref = None
for mb in mbs:
    os.environ["IGA2L_S3D_ZCHUNK_MB"] = mb
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
    same = torch.equal(x, ref)
    ms = 0.0
    for _ in range(3):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1) / 3
    print(f"{name} IGA2L_S3D_ZCHUNK_MB={mb}: sweep {ms:.2f} ms; bitwise equal to the first: {same}", flush=True)
    del g
