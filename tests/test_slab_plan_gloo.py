"""Multi-process (world_size 2 and 3, gloo, CPU) test of the slab decomposition the library uses
for nranks > 1: the plan comes from the library (`iga2l_host_slab_plan`), the block
arithmetic from the oracle, the halo exchanges are real torch.distributed send/recv.  Each rank
keeps only its stored planes [za, zb) (everything else is NaN, so a read outside the halo would
poison the result); the gathered owned planes must equal the global multicolour sweep BITWISE.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.multiproc

CASES = [  # (d, p, m, s, world)
    (2, 3, 20, 3, 2),
    (2, 5, 24, 5, 3),
    (2, 8, 36, 7, 2),
    (3, 3, 10, 3, 2),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, outdir):
    import torch.distributed as dist
    import torch

    import paper_2009_01499_b200 as pkg
    from oracle.assembly import stiffness
    from oracle.schwarz import Schwarz, colour_of
    from synthetic_inputs import initial_guess, random_rhs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, p, m, s, _ = case
    n1 = m + p - 2
    plane = n1 ** (d - 1)
    plan = pkg.host_slab_plan(d, p, s, m, world, rank)
    assert plan["feasible"] == 1
    z0, z1, za, zb, clo, chi, H = (plan[k] for k in ("z0", "z1", "za", "zb", "c_lo", "c_hi", "H"))
    A = stiffness(p, m, d)
    sm = Schwarz(A, n1, d, s, p, order="multicolour")
    b = random_rhs(n1 ** d)
    xg = initial_guess(n1 ** d)
    # local copy: only the stored planes are valid
    x = np.full(n1 ** d, np.nan)
    x[za * plane:zb * plane] = xg[za * plane:zb * plane]
    bl = np.full(n1 ** d, np.nan)
    bl[za * plane:zb * plane] = b[za * plane:zb * plane]
    D = s + p
    per_class = D ** (d - 1)

    def exchange():
        reqs = []
        if rank > 0:   # own bottom H planes -> rank-1's upper halo; receive my lower halo
            reqs.append(dist.isend(torch.from_numpy(x[z0 * plane:(z0 + H) * plane].copy()), rank - 1))
            lo = torch.empty(H * plane, dtype=torch.float64)
            reqs.append(dist.irecv(lo, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(x[(z1 - H) * plane:z1 * plane].copy()), rank + 1))
            hi = torch.empty(H * plane, dtype=torch.float64)
            reqs.append(dist.irecv(hi, rank + 1))
        for r in reqs:
            r.wait()
        if rank > 0:
            x[za * plane:z0 * plane] = lo.numpy()
        if rank < world - 1:
            x[z1 * plane:zb * plane] = hi.numpy()

    by_colour = {}
    for c in sm.seq:
        by_colour.setdefault(colour_of(c, D), []).append(c)
    for zc in range(D):
        if zc > 0:
            exchange()
        for k in range(per_class):
            for c in by_colour.get(zc * per_class + k, []):
                if clo <= c[d - 1] < chi:          # last-axis centre handled by this rank
                    sm.step(x, bl, c)
    exchange()
    np.save(os.path.join(outdir, f"slab{rank}.npy"), x[z0 * plane:z1 * plane])
    if rank == 0:
        ref = sm.sweep(xg.copy(), b)
        np.save(os.path.join(outdir, "ref.npy"), ref)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES, ids=[f"d{c[0]}p{c[1]}m{c[2]}s{c[3]}w{c[4]}" for c in CASES])
def test_slab_sweep_equals_global_sweep(case, tmp_path):
    import torch.multiprocessing as mp
    import __graft_entry__
    __graft_entry__.build()
    world = case[4]
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    ref = np.load(tmp_path / "ref.npy")
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)])
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref)
