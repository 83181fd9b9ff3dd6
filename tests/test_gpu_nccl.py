"""Two-process NCCL run of the slab-partitioned iteration: one slab per process and GPU,
halos and the coarse-defect reduction over NCCL (the ncclUniqueId from rank 0's library broadcast over
torch.distributed), against the single-domain CUDA path on one device.  Needs >= 2 GPUs (skipped
otherwise: the round-end boxes have one; the same schedule runs on one device in test_gpu_slabs.py)."""
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)

CASES = [("2d_p3", 2, 3, 1, 48, 3), ("3d_p3", 3, 3, 1, 20, 3), ("3d_p5_q2", 3, 5, 2, 32, 5)]


def _worker(rank, world, port, case, out):
    import torch.distributed as dist
    import paper_2009_01499_b200 as pkg
    from synthetic_inputs import initial_guess, random_rhs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, d, p, q, m, s = case
    nid = [pkg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(nid, src=0)
    st = torch.cuda.Stream()
    ctx = pkg.Context(d, p, q, m, s, coarse_mode=pkg.COARSE_VCYCLE, coarse_h_factor=2, stream=st.cuda_stream,
                      nranks=world, rank=rank, nccl_id=nid[0])
    n1 = m + p - 2
    plane = n1 ** (d - 1)
    sl = slice(ctx.z0 * plane, ctx.z1 * plane)
    b = torch.tensor(random_rhs(n1 ** d)[sl], device="cuda")
    x = torch.tensor(initial_guess(n1 ** d)[sl], device="cuda")
    hist = np.zeros(4)
    ctx.iterate(b, x, 3, hist)
    torch.cuda.synchronize()
    np.save(os.path.join(out, f"x{rank}.npy"), x.cpu().numpy())
    np.save(os.path.join(out, f"h{rank}.npy"), hist)
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_two_process_nccl_slabs_match_single_domain(case):
    import torch.multiprocessing as mp
    import paper_2009_01499_b200 as pkg
    from synthetic_inputs import initial_guess, random_rhs
    _, d, p, q, m, s = case
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(2, 29500 + os.getpid() % 1000, case, out), nprocs=2, join=True)
        xs = [np.load(os.path.join(out, f"x{r}.npy")) for r in range(2)]
        h0 = np.load(os.path.join(out, "h0.npy"))
    n1 = m + p - 2
    ctx = pkg.Context(d, p, q, m, s, coarse_mode=pkg.COARSE_VCYCLE, coarse_h_factor=2)
    b = torch.tensor(random_rhs(n1 ** d), device="cuda")
    x = torch.tensor(initial_guess(n1 ** d), device="cuda")
    hist = np.zeros(4)
    ctx.iterate(b, x, 3, hist)
    torch.cuda.synchronize()
    ref = x.cpu().numpy()
    got = np.concatenate(xs)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.allclose(h0, hist, rtol=1e-10)
