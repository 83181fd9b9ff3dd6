"""GPU test of the slab-decomposed path on one device: nranks slabs held by one
context (rank = -1), halos exchanged by device copies, partial restrictions summed in a fixed order.
The kernels and the schedule are exactly those of the NCCL path (one slab per process); only the
transport differs.  Compared with the single-domain CUDA path and with the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2009_01499_b200 as pkg  # noqa: E402
from oracle.twolevel import TwoLevel  # noqa: E402
from synthetic_inputs import initial_guess, random_rhs  # noqa: E402

DEV = torch.device("cuda:0")
STREAM = torch.cuda.Stream(DEV)


@pytest.fixture(autouse=True)
def _on_stream():
    with torch.cuda.stream(STREAM):
        yield
    torch.cuda.synchronize()


CASES = [  # (name, d, p, q, m, s, coarse, h_factor, nranks)
    ("C1_R3", 2, 2, 1, 16, 3, "exact", 1, 3),
    ("2d_p3_R2", 2, 3, 1, 48, 3, "vcycle", 2, 2),
    ("2d_p3_R4", 2, 3, 1, 48, 3, "vcycle", 2, 4),
    ("2d_p5_R3", 2, 5, 1, 64, 5, "vcycle", 2, 3),
    ("2d_p8_q2_R2", 2, 8, 2, 64, 7, "vcycle", 2, 2),
    ("3d_p3_R2", 3, 3, 1, 20, 3, "vcycle", 2, 2),
    ("3d_p3_R4", 3, 3, 1, 20, 3, "vcycle", 2, 4),
    ("3d_p5_q2_R2", 3, 5, 2, 16, 5, "vcycle", 2, 2),
]


def ctx_for(d, p, q, m, s, coarse, hf, nranks=1, rank=0):
    return pkg.Context(d, p, q, m, s, coarse_mode=pkg.COARSE_EXACT if coarse == "exact" else pkg.COARSE_VCYCLE,
                       coarse_h_factor=hf, stream=STREAM.cuda_stream, nranks=nranks, rank=rank)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_slabs_match_single_domain_and_oracle(case):
    name, d, p, q, m, s, coarse, hf, R = case
    one = ctx_for(d, p, q, m, s, coarse, hf)
    sl = ctx_for(d, p, q, m, s, coarse, hf, nranks=R, rank=-1)
    N = one.N
    b, x0 = random_rhs(N), initial_guess(N)
    bg = torch.tensor(b, device=DEV)
    x1, x2 = torch.tensor(x0, device=DEV), torch.tensor(x0, device=DEV)
    h1, h2 = np.zeros(6), np.zeros(6)
    one.iterate(bg, x1, 5, h1)
    sl.iterate(bg, x2, 5, h2)
    torch.cuda.synchronize()
    a1, a2 = x1.cpu().numpy(), x2.cpu().numpy()
    assert np.linalg.norm(a2 - a1) <= 1e-12 * np.linalg.norm(a1)
    assert np.allclose(h2, h1, rtol=1e-9, atol=1e-12 * h1[0])
    if N <= 20000:
        ora = TwoLevel(d, p, q, m, s=s, coarse=coarse, h_factor=hf)
        xo = x0.copy()
        for _ in range(5):
            ora.iterate(xo, b)
        assert np.linalg.norm(a2 - xo) <= 1e-10 * np.linalg.norm(xo)
    # apply and the residual norm through the slab path
    y1, y2 = torch.empty_like(bg), torch.empty_like(bg)
    one.apply(x1, y1)
    sl.apply(x1, y2)
    torch.cuda.synchronize()
    assert torch.allclose(y1, y2, rtol=0, atol=1e-13 * float(y1.abs().max()))
    assert abs(sl.residual_norm(bg, x1) - one.residual_norm(bg, x1)) <= 1e-12 * one.residual_norm(bg, x1)


def test_slab_solve_iterations_match():
    d, p, q, m, s = 2, 4, 1, 64, 3
    one = ctx_for(d, p, q, m, s, "vcycle", 2)
    sl = ctx_for(d, p, q, m, s, "vcycle", 2, nranks=3, rank=-1)
    b = torch.empty(one.N, dtype=torch.float64, device=DEV)
    one.rhs_sine(b)
    x1 = torch.tensor(initial_guess(one.N), device=DEV)
    x2 = x1.clone()
    it1, r1, ok1 = one.solve(b, x1, 1e-8, 60)
    it2, r2, ok2 = sl.solve(b, x2, 1e-8, 60)
    assert ok1 and ok2 and it1 == it2


def test_slab_errors():
    with pytest.raises(pkg.IgaError):        # slabs thinner than the halo s - 1 + p
        ctx_for(2, 8, 2, 16, 7, "vcycle", 2, nranks=4, rank=-1)
    with pytest.raises(pkg.IgaError):        # NCCL rank without an id
        ctx_for(2, 3, 1, 48, 3, "vcycle", 2, nranks=2, rank=0)
