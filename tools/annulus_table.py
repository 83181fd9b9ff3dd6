"""Table 5 protocol on the GPU (quarter annulus): for every grid m^2 (m = 32..256) and degree p = 3..8
with the paper's block sizes, DS (exact second level) and MG (one V(1,1)), both at H = 2h:
iterations to ||r|| <= 1e-8 ||r_0|| from x_0 ~ U[-1,1] seed 0 on the paper's f, and the device time per
iteration (CUDA events around graph replays of iga2l_iterate).  The paper's counts are printed beside
(context: its three-colour order is not available, readings A4/A21)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_01499_b200 as pkg  # noqa: E402
from synthetic_inputs import initial_guess  # noqa: E402

PAPER = {  # Table 5: (DS, MG) per grid, p = 3..8
    32: [(5, 5), (8, 8), (4, 4), (6, 6), (3, 3), (4, 4)],
    64: [(5, 7), (8, 8), (4, 5), (6, 6), (4, 4), (5, 5)],
    128: [(6, 8), (7, 8), (4, 6), (6, 6), (4, 5), (5, 5)],
    256: [(6, 9), (8, 8), (4, 6), (6, 6), (4, 6), (5, 6)],
}
BLOCK = {3: 3, 4: 3, 5: 5, 6: 5, 7: 7, 8: 7}

dev = torch.device("cuda:0")
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
print(f"{'grid':>6} {'p':>2} | {'DS it':>5} {'MG it':>5} | paper DS MG | {'DS us/it':>9} {'MG us/it':>9}")
for m in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else sorted(PAPER))]:
    for i, p in enumerate(range(3, 9)):
        res = []
        for mode in (pkg.COARSE_EXACT, pkg.COARSE_VCYCLE):
            ctx = pkg.Context(2, p, 2, m, BLOCK[p], coarse_mode=mode, stream=st.cuda_stream, geometry="annulus")
            b = torch.empty(ctx.N, dtype=torch.float64, device=dev)
            ctx.rhs(b)
            x0 = torch.tensor(initial_guess(ctx.N), device=dev)
            it, rr, ok = ctx.solve(b, x0.clone(), rtol=1e-8, maxit=100)
            x = x0.clone()
            ctx.iterate(b, x, 3)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            ctx.iterate(b, x, 20)
            e1.record(st)
            torch.cuda.synchronize()
            res.append((it if ok else -1, 1e3 * e0.elapsed_time(e1) / 20))
            ctx.close()
        pd, pm = PAPER[m][i]
        print(f"{m:>4}^2 {p:>2} | {res[0][0]:>5} {res[1][0]:>5} | {pd:>5} {pm:>3} | {res[0][1]:>9.1f} {res[1][1]:>9.1f}",
              flush=True)
