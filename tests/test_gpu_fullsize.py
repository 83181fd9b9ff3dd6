"""GPU parity at full BASELINE sizes (and at the 3D shapes the survey names), against the matrix-free
oracle ``oracle.kron.KronTwoLevel`` (pinned to the assembled sequential ``TwoLevel`` in
tests/test_oracle_kron.py), element by element, in the launch configuration bench.py times.

North-star bars (BASELINE.json): ||x_gpu - x_oracle|| / ||x_oracle|| <= 1e-10 after 5 iterations of
Algorithm 1; measured convergence factor within 2% of the oracle's (P:311 protocol:
b = 0, random x_0, geometric mean of the last residual ratios).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2009_01499_b200 as pkg  # noqa: E402
from oracle.kron import KronOperator, KronTwoLevel  # noqa: E402
from oracle.multigrid import QHierarchy  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess, random_rhs  # noqa: E402

DEV = torch.device("cuda:0")
STREAM = torch.cuda.Stream(DEV)


@pytest.fixture(autouse=True)
def _on_stream():
    with torch.cuda.stream(STREAM):
        yield
    torch.cuda.synchronize()


def cu(a):
    return torch.tensor(a, dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def make_ctx(d, p, q, m, s, coarse="vcycle", hf=2):
    return pkg.Context(d, p, q, m, s, coarse_mode=pkg.COARSE_EXACT if coarse == "exact" else pkg.COARSE_VCYCLE,
                       coarse_h_factor=hf, stream=STREAM.cuda_stream)


# (name, d, p, q, m, s, factor iterations, ratios averaged): C2 at its full size; C4 / C5 shapes at the
# sizes the survey's parity runs name: m = 48 (C4 shape), m = 32 (C5 shape, q = 2: the
# second level m_c = 16 runs a real 3D q = 2 V(1,1) with one smoothing level above the direct solve).
FULL = [("C2p3", 2, 3, 1, 256, 3, 25, 10), ("C2p4", 2, 4, 1, 256, 3, 25, 10), ("C2p5", 2, 5, 1, 256, 5, 25, 10),
        ("C4_m48", 3, 3, 1, 48, 3, 15, 8), ("C5_m32", 3, 5, 2, 32, 5, 12, 6)]
_oracles = {}


def oracle(name, d, p, q, m, s):
    if name not in _oracles:
        _oracles.clear()                                 # one at a time (C5_m32 keeps 5.4 GB of inverses)
        _oracles[name] = KronTwoLevel(d, p, q, m, s)
    return _oracles[name]


@pytest.mark.parametrize("cfg", FULL, ids=[c[0] for c in FULL])
def test_five_iterations_full_size(cfg):
    name, d, p, q, m, s, _, _ = cfg
    if name.startswith("C2"):
        c = CONFIGS[name]
        assert (c["d"], c["p"], c["q"], c["m"], c["s"]) == (d, p, q, m, s)
    ora = oracle(name, d, p, q, m, s)
    ctx = make_ctx(d, p, q, m, s)
    assert ctx.N == ora.N
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xg = cu(x0)
    hist = np.zeros(6)
    ctx.iterate(cu(b), xg, iters=5, res_hist=hist)
    xo = x0.copy()
    ho = [np.linalg.norm(b - ora.A.apply(xo))]
    for _ in range(5):
        ora.iterate(xo, b)
        ho.append(np.linalg.norm(b - ora.A.apply(xo)))
    rel = np.linalg.norm(host(xg) - xo) / np.linalg.norm(xo)
    assert rel <= 1e-10, rel
    assert np.all(np.abs(hist - ho) <= 1e-8 * np.asarray(ho) + 1e-12 * ho[0]), (hist, ho)


# The remaining 2D/3D BASELINE configs at their FULL sizes (SURVEY §8(d) parity plan: C1-C4 full):
# the oracle needs minutes per iteration here (C4: ~85 s, 16 cores), so these run on request
# (IGA2L_SLOW_PARITY=1; record: profiles/tests_gpu_slow_parity_r02.txt), not in the default GPU suite.
SLOW = [("C4", 3, 3, 1, 128, 3), ("C3", 2, 8, 2, 1024, 7)]


@pytest.mark.skipif(not __import__("os").environ.get("IGA2L_SLOW_PARITY"), reason="slow: IGA2L_SLOW_PARITY=1")
@pytest.mark.parametrize("cfg", SLOW, ids=[c[0] for c in SLOW])
def test_five_iterations_full_config(cfg):
    name, d, p, q, m, s = cfg
    if name in CONFIGS:
        c = CONFIGS[name]
        assert (c["d"], c["p"], c["q"], c["m"], c["s"]) == (d, p, q, m, s)
    _oracles.clear()
    ora = KronTwoLevel(d, p, q, m, s)
    ctx = make_ctx(d, p, q, m, s)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xg = cu(x0)
    hist = np.zeros(6)
    ctx.iterate(cu(b), xg, iters=5, res_hist=hist)
    xo = x0.copy()
    ho = [np.linalg.norm(b - ora.A.apply(xo))]
    for _ in range(5):
        ora.iterate(xo, b)
        ho.append(np.linalg.norm(b - ora.A.apply(xo)))
    rel = np.linalg.norm(host(xg) - xo) / np.linalg.norm(xo)
    print(f"{name}: ||x_gpu - x_oracle|| / ||x_oracle|| after 5 iterations = {rel:.3e}; residuals {hist}")
    assert rel <= 1e-10, rel
    assert np.all(np.abs(hist - ho) <= 1e-8 * np.asarray(ho) + 1e-12 * ho[0]), (hist, ho)


@pytest.mark.parametrize("cfg", FULL, ids=[c[0] for c in FULL])
def test_convergence_factor_full_size(cfg):
    name, d, p, q, m, s, iters, last = cfg
    ora = oracle(name, d, p, q, m, s)
    ctx = make_ctx(d, p, q, m, s)
    x0 = initial_guess(ctx.N)
    rate_o, _ = ora.rate(x0, iters=iters, last=last)
    hist = np.zeros(iters + 1)
    ctx.iterate(cu(np.zeros(ctx.N)), cu(x0), iters=iters, res_hist=hist)
    ratios = hist[1:] / hist[:-1]
    rate_g = float(np.exp(np.mean(np.log(ratios[-last:]))))
    assert abs(rate_g - rate_o) <= 0.02 * rate_o, (rate_g, rate_o)


# ---- the second level alone at full size, against QHierarchy.vcycle ----
VC = [(1, 128, 2, 3, 3), (1, 64, 3, 3, 3), (2, 512, 2, 8, 7), (2, 32, 3, 5, 5), (2, 64, 3, 5, 5), (2, 128, 3, 5, 5)]


@pytest.mark.parametrize("q,m,d,p,s", VC, ids=["C2", "C4", "C3", "3d_q2_m32", "3d_q2_m64", "C5"])
def test_vcycle_full_size(q, m, d, p, s):
    H = QHierarchy(q, m, d)
    n = H.levels[0]["n"]
    ctx = make_ctx(d, p, q, 2 * m, s)      # aggressive second level of a fine m = 2 m context is this q-level
    assert ctx.Nc == n ** d
    dq = random_rhs(ctx.Nc, seed=5)
    e = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.coarse_solve(cu(dq), e)
    ref = H.vcycle(dq)
    assert np.abs(host(e) - ref).max() <= 1e-11 * np.abs(ref).max()


@pytest.mark.parametrize("cs", [2, 4, 8, 16])
@pytest.mark.parametrize("m", [32, 64], ids=["mc16", "mc32"])
def test_vcycle_smem_spread_3d_q2(m, cs, monkeypatch):
    """The 3D q = 2 second level with its first level SPREAD over a cluster of cs CTAs (DSMEM halos)."""
    monkeypatch.setenv("IGA2L_VC_FORCE_CS", str(cs))
    H = QHierarchy(2, m // 2, 3)
    ctx = make_ctx(3, 5, 2, m, 5)
    inf = ctx.info()
    if m == 32 and cs <= 8:                # >= 2 rows per CTA and it fits: the DSMEM spread path must run
        assert (inf.vc_smem_level, inf.vc_smem_cs) == (0, cs), (inf.vc_smem_level, inf.vc_smem_cs)
    dq = random_rhs(ctx.Nc, seed=3)
    e = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.coarse_solve(cu(dq), e)
    ref = H.vcycle(dq)
    assert np.abs(host(e) - ref).max() <= 1e-11 * np.abs(ref).max()


# ---- C3 transfers at full size (the separable 32x32-tile kernel bench.py runs) and that kernel forced
# at small sizes, against the oracle's Kronecker R ----
@pytest.mark.parametrize("force", [None, "32"], ids=["auto", "sep32"])
@pytest.mark.parametrize("d,p,q,m,s", [(2, 8, 2, 1024, 7), (2, 8, 2, 32, 7), (2, 3, 1, 48, 3), (2, 5, 1, 40, 5)],
                         ids=["C3", "p8_m32", "p3_m48", "p5_m40"])
def test_transfers_2d(d, p, q, m, s, force, monkeypatch):
    if force:
        monkeypatch.setenv("IGA2L_TRANSFER_SEP", force)
    ctx = make_ctx(d, p, q, m, s)
    ora = KronTwoLevel.__new__(KronTwoLevel)                       # transfers + operator only (no V-cycle setup)
    from oracle.transfer import degree_restriction_1d, mesh_prolongation_1d
    import scipy.sparse as sp
    R1 = mesh_prolongation_1d(q, m // 2).T @ degree_restriction_1d(p, q, m)
    ora.d, ora.n1, ora.nc1 = d, m + p - 2, R1.shape[0]
    ora.R1, ora.R1T = sp.csr_matrix(R1), sp.csr_matrix(R1.T)
    A = KronOperator(p, m, d)
    b, x = random_rhs(ctx.N, seed=8), initial_guess(ctx.N, seed=9)
    dq = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.defect_restrict(cu(b), cu(x), dq)
    ref = ora.restrict(b - A.apply(x))
    absA = KronOperator(p, m, d)                                   # |A| |x| bound: the terms that cancel
    absA.K, absA.M = abs(absA.K), abs(absA.M)
    ora_abs = KronTwoLevel.__new__(KronTwoLevel)
    ora_abs.d, ora_abs.n1, ora_abs.R1 = d, ora.n1, abs(ora.R1)
    scale = ora_abs.restrict(np.abs(b) + absA.apply(np.abs(x))).max()
    assert np.abs(host(dq) - ref).max() <= 1e-13 * scale
    e = random_rhs(ctx.Nc, seed=10)
    xp = cu(x)
    ctx.prolong_add(cu(e), xp)
    ref = x + ora.prolong(e)
    assert np.abs(host(xp) - ref).max() <= 1e-13 * np.abs(ref).max()
