"""GPU parity of the quarter-annulus NURBS workload against
``oracle.annulus.AnnulusTwoLevel`` (2D element-by-element assembly on the exact geometry; pinned in
tests/test_oracle_annulus.py).  The CUDA path runs the SAME kernels as the square with per-axis weighted
1D tables (A = My ⊗ Kx + Ky ⊗ Mx, exact on this orthogonal map) and per-axis transfers.

Bars as tests/test_gpu_parity.py: phase outputs max |gpu - oracle| <= 1e-11 max |oracle| (the oracle's
2D assembly and the 1D tables agree to ~1e-13, see test_tensor_structure_on_the_map); 5 iterations
||x_gpu - x_oracle|| / ||x_oracle|| <= 1e-10; Table 5 protocol iteration counts equal.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2009_01499_b200 as pkg  # noqa: E402
from oracle import annulus as an  # noqa: E402
from synthetic_inputs import initial_guess, random_rhs  # noqa: E402

DEV = torch.device("cuda:0")
STREAM = torch.cuda.Stream(DEV)


@pytest.fixture(autouse=True)
def _on_stream():
    with torch.cuda.stream(STREAM):
        yield
    torch.cuda.synchronize()


# (name, p, m, s, coarse): DMMA colour kernel for (p, s) in the paper's pairs, the generic kernel for
# (3, 5); V(1,1) with two levels at m = 32 (m_c = 16 -> 8), exact dense / FD second level.
CASES = [("p3_vc", 3, 32, 3, "vcycle"), ("p2_ex", 2, 16, 3, "exact"), ("p5_vc", 5, 32, 5, "vcycle"),
         ("p8_ex", 8, 16, 7, "exact"), ("p3_s5_generic", 3, 16, 5, "vcycle"), ("p4_ex_fd", 4, 32, 3, "exact_fd")]
_or = {}


def oracle(p, m, s, coarse):
    key = (p, m, s, coarse)
    if key not in _or:
        _or.clear()
        _or[key] = an.AnnulusTwoLevel(p, m, s, coarse="vcycle" if coarse == "vcycle" else "exact")
    return _or[key]


def ctx_for(p, m, s, coarse, monkeypatch):
    if coarse == "exact_fd":
        monkeypatch.setenv("IGA2L_COARSE_FD", "1")
    return pkg.Context(2, p, 2, m, s, coarse_mode=pkg.COARSE_VCYCLE if coarse == "vcycle" else pkg.COARSE_EXACT,
                       stream=STREAM.cuda_stream, geometry="annulus")


def cu(a):
    return torch.tensor(a, dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def close(got, ref, tol=1e-11):
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err <= tol, err


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_phases(case, monkeypatch):
    _, p, m, s, coarse = case
    ora = oracle(p, m, s, coarse)
    ctx = ctx_for(p, m, s, coarse, monkeypatch)
    assert (ctx.N, ctx.Nc) == (ora.N, ora.Nc)
    x, b = initial_guess(ctx.N, seed=4), random_rhs(ctx.N, seed=5)
    y = torch.empty(ctx.N, dtype=torch.float64, device=DEV)
    ctx.apply(cu(x), y)
    close(host(y), ora.A @ x, 1e-12)
    xs = cu(x)
    ctx.sweep(cu(b), xs)
    xo = x.copy()
    ora.smoother.sweep(xo, b)
    close(host(xs), xo)
    dq = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.defect_restrict(cu(b), cu(x), dq)
    close(host(dq), ora.R @ (b - ora.A @ x))
    d = random_rhs(ctx.Nc, seed=6)
    e = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.coarse_solve(cu(d), e)
    close(host(e), ora._csolve(d))
    xp = cu(x)
    ctx.prolong_add(cu(d), xp)
    close(host(xp), x + ora.RT @ d)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_five_iterations(case, monkeypatch):
    _, p, m, s, coarse = case
    ora = oracle(p, m, s, coarse)
    ctx = ctx_for(p, m, s, coarse, monkeypatch)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xg = cu(x0)
    hist = np.zeros(6)
    ctx.iterate(cu(b), xg, iters=5, res_hist=hist)
    xo = x0.copy()
    ho = [np.linalg.norm(b - ora.A @ xo)]
    for _ in range(5):
        ora.iterate(xo, b)
        ho.append(np.linalg.norm(b - ora.A @ xo))
    assert np.linalg.norm(host(xg) - xo) / np.linalg.norm(xo) <= 1e-10
    assert np.all(np.abs(hist - ho) <= 1e-8 * np.asarray(ho) + 1e-12 * ho[0]), (hist, ho)


@pytest.mark.parametrize("p,m", [(3, 16), (6, 8)])
def test_rhs(p, m):
    ctx = pkg.Context(2, p, 2, m, 3 if p <= 4 else 5, stream=STREAM.cuda_stream, geometry="annulus")
    b = torch.empty(ctx.N, dtype=torch.float64, device=DEV)
    ctx.rhs(b)
    close(host(b), an.assemble(p, m, want=("b",))["b"], 1e-13)


@pytest.mark.parametrize("p,s", [(3, 3), (5, 5)])
def test_table5_protocol_iterations(p, s):
    """Iterations to ||r|| <= 1e-8 ||r_0|| from a random x_0 on the paper's f (Table 5), DS and MG:
    the GPU count equals the oracle's (the paper's own counts are context: its colour order, A4/A21)."""
    m = 32
    for coarse in ("exact", "vcycle"):
        ora = an.AnnulusTwoLevel(p, m, s, coarse=coarse)
        ctx = pkg.Context(2, p, 2, m, s, coarse_mode=pkg.COARSE_EXACT if coarse == "exact" else pkg.COARSE_VCYCLE,
                          stream=STREAM.cuda_stream, geometry="annulus")
        x0 = initial_guess(ctx.N)
        _, it_o, _ = ora.solve(ora.b, x0, rtol=1e-8)
        b = torch.empty(ctx.N, dtype=torch.float64, device=DEV)
        ctx.rhs(b)
        it_g, rr, ok = ctx.solve(b, cu(x0), rtol=1e-8, maxit=100)
        assert ok and rr <= 1e-8
        assert it_g == it_o, (coarse, it_g, it_o)


def test_annulus_rejects_unsupported():
    for args in [dict(dim=3, q=2), dict(dim=2, q=1)]:
        with pytest.raises(pkg.IgaError):
            pkg.Context(args["dim"], 3, args["q"], 16, 3, stream=STREAM.cuda_stream, geometry="annulus")
