"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded inputs.

Bars (BASELINE.json north_star):
  * operator/phase outputs (apply, rhs, one sweep, defect+restriction, coarse solve, prolongation):
    max |gpu - oracle| <= 1e-12 * max |oracle| (fp64, summation order differs);
  * 5 two-level iterations: ||x_gpu - x_oracle|| / ||x_oracle|| <= 1e-10;
  * measured convergence factor within 2% of the oracle's.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2009_01499_b200 as pkg  # noqa: E402
from oracle.assembly import load_sine  # noqa: E402
from oracle.sampled import RowOracle  # noqa: E402
from oracle.twolevel import TwoLevel  # noqa: E402
from synthetic_inputs import CONFIGS, initial_guess, random_rhs  # noqa: E402

DEV = torch.device("cuda:0")
STREAM = torch.cuda.Stream(DEV)      # torch ops and library calls share this one stream


@pytest.fixture(autouse=True)
def _on_stream():
    with torch.cuda.stream(STREAM):
        yield
    torch.cuda.synchronize()

# (name, d, p, q, m, s, coarse, h_factor): parity sizes the oracle finishes in seconds, each with
# several tiles/colours and a ragged tail (n1 not a multiple of D nor of the tile sizes).
PAR = [
    ("C1", 2, 2, 1, 16, 3, "exact", 1),
    ("2d_p1", 2, 1, 1, 16, 3, "exact", 1),
    ("2d_p3_vc", 2, 3, 1, 48, 3, "vcycle", 2),
    ("2d_p4_vc", 2, 4, 1, 40, 3, "vcycle", 2),
    ("2d_p5_vc", 2, 5, 1, 32, 5, "vcycle", 2),
    ("2d_p8_q2", 2, 8, 2, 32, 7, "vcycle", 2),
    ("2d_p2_sameh_vc", 2, 2, 1, 32, 3, "vcycle", 1),
    ("3d_p3_vc", 3, 3, 1, 20, 3, "vcycle", 2),
    ("3d_p5_q2", 3, 5, 2, 10, 5, "vcycle", 2),
    ("2d_tiny", 2, 2, 1, 3, 3, "exact", 1),
]

_oracles = {}


def oracle_for(name, d, p, q, m, s, coarse, hf):
    key = (d, p, q, m, s, coarse, hf)
    if key not in _oracles:
        _oracles[key] = TwoLevel(d, p, q, m, s=s, coarse=coarse, h_factor=hf, order="multicolour")
    return _oracles[key]


def make_ctx(d, p, q, m, s, coarse, hf, **kw):
    return pkg.Context(d, p, q, m, s, coarse_mode=pkg.COARSE_EXACT if coarse == "exact" else pkg.COARSE_VCYCLE,
                       coarse_h_factor=hf, stream=STREAM.cuda_stream, **kw)


def cu(a):
    return torch.tensor(a, dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def close(got, ref, tol=1e-12):
    scale = max(np.abs(ref).max(), 1e-300)
    err = np.abs(got - ref).max() / scale
    assert err <= tol, f"max rel err {err:.3e} > {tol:.1e}"


@pytest.mark.parametrize("cfg", PAR, ids=[c[0] for c in PAR])
def test_apply_and_rhs(cfg):
    name, d, p, q, m, s, coarse, hf = cfg
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    x = initial_guess(ctx.N)
    y = torch.empty(ctx.N, dtype=torch.float64, device=DEV)
    ctx.apply(cu(x), y)
    close(host(y), ora.A @ x, 1e-13)
    b = torch.empty_like(y)
    ctx.rhs_sine(b)
    close(host(b), load_sine(p, m, d), 1e-14)


@pytest.mark.parametrize("cfg", PAR, ids=[c[0] for c in PAR])
def test_one_sweep_and_phases(cfg):
    name, d, p, q, m, s, coarse, hf = cfg
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xg = cu(x0)
    ctx.sweep(cu(b), xg)
    xo = ora.smoother.sweep(x0.copy(), b)
    # one sweep = N block solves in sequence; FD vs Cholesky local solves differ by ~κ(A_B)·eps
    close(host(xg), xo, 1e-11)
    # defect + restriction
    dq = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.defect_restrict(cu(b), cu(xo), dq)
    dqo = ora.R @ (b - ora.A @ xo)
    # b - A x cancels (the sweep just reduced it): scale by the terms, not by the result
    scale = np.abs(ora.R) @ (np.abs(b) + np.abs(ora.A) @ np.abs(xo))
    assert np.abs(host(dq) - dqo).max() <= 1e-13 * scale.max()
    # second-level solve (exact or one V(1,1))
    e = torch.empty_like(dq)
    ctx.coarse_solve(cu(dqo), e)
    eo = ora._csolve(dqo)
    close(host(e), eo, 1e-11)
    # prolongation x += R^T e
    xp = cu(xo)
    ctx.prolong_add(cu(eo), xp)
    close(host(xp), xo + ora.RT @ eo)


@pytest.mark.parametrize("cfg", PAR, ids=[c[0] for c in PAR])
def test_five_iterations(cfg):
    name, d, p, q, m, s, coarse, hf = cfg
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xg = cu(x0)
    hist = np.zeros(6)
    ctx.iterate(cu(b), xg, iters=5, res_hist=hist)
    xo = x0.copy()
    ho = [np.linalg.norm(b - ora.A @ xo)]
    for _ in range(5):
        ora.iterate(xo, b)
        ho.append(np.linalg.norm(b - ora.A @ xo))
    rel = np.linalg.norm(host(xg) - xo) / np.linalg.norm(xo)
    assert rel <= 1e-10, rel
    # residual norms agree until they reach the rounding floor of the (converged) iterate
    assert np.all(np.abs(hist - ho) <= 1e-8 * np.asarray(ho) + 1e-12 * ho[0]), (hist, ho)


def test_iters_zero_is_noop_and_deterministic():
    ctx = make_ctx(2, 3, 1, 48, 3, "vcycle", 2)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    x = x0.clone()
    ctx.iterate(b, x, iters=0)
    assert torch.equal(x, x0)
    x1, x2 = x0.clone(), x0.clone()
    ctx.iterate(b, x1, iters=3)
    ctx.iterate(b, x2, iters=3)
    assert torch.equal(x1, x2)                      # bitwise, no atomics on value paths
    # graph replay == eager launches
    ctx_e = make_ctx(2, 3, 1, 48, 3, "vcycle", 2, use_graph=False)
    x3 = x0.clone()
    ctx_e.iterate(b, x3, iters=3)
    assert torch.equal(x1, x3)


def test_host_pointers_match_device():
    ctx = make_ctx(2, 4, 1, 40, 3, "vcycle", 2)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xd = cu(x0)
    ctx.iterate(cu(b), xd, iters=2)
    xh = x0.copy()
    ctx.iterate(b, xh, iters=2)                    # numpy (host) buffers, staged by the library
    assert np.array_equal(host(xd), xh)


@pytest.mark.parametrize("cfg", [PAR[0], PAR[3], PAR[7]], ids=["C1", "2d_p4", "3d_p3"])
def test_convergence_factor_within_2pct(cfg):
    name, d, p, q, m, s, coarse, hf = cfg
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    x0 = initial_guess(ctx.N)
    rate_o, _ = ora.rate(x0, iters=25)
    hist = np.zeros(26)
    ctx.iterate(cu(np.zeros(ctx.N)), cu(x0), iters=25, res_hist=hist)
    ratios = hist[1:] / hist[:-1]
    rate_g = float(np.exp(np.mean(np.log(ratios[-10:]))))
    assert abs(rate_g - rate_o) <= 0.02 * rate_o, (rate_g, rate_o)


@pytest.mark.parametrize("cfg", [PAR[0], PAR[2]], ids=["C1", "2d_p3"])
def test_solve_matches_oracle(cfg):
    name, d, p, q, m, s, coarse, hf = cfg
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    b = load_sine(p, m, d)
    x0 = initial_guess(ctx.N)
    xg = cu(x0)
    it, rr, ok = ctx.solve(cu(b), xg, rtol=1e-8, maxit=50)
    xo, ito, ho = ora.solve(b, x0, rtol=1e-8)
    assert ok and it == ito
    assert rr <= 1e-8
    assert np.linalg.norm(host(xg) - xo) <= 1e-9 * np.linalg.norm(xo)


# ---- full BASELINE sizes, in the launch configuration bench.py times: sampled outputs ----
FULL = ["C2p3", "C2p4", "C2p5", "C3", "C4", "C5"]


@pytest.mark.parametrize("name", FULL)
def test_full_size_sampled(name):
    cfg = CONFIGS[name]
    d, p, q, m, s = cfg["d"], cfg["p"], cfg["q"], cfg["m"], cfg["s"]
    ctx = make_ctx(d, p, q, m, s, cfg["coarse"], cfg["h_factor"])
    N, n1, D = ctx.N, ctx.n1, s + p
    ro = RowOracle(p, m, d)
    rng = np.random.default_rng(7)
    x0, b = initial_guess(N), random_rhs(N)
    # apply on sampled rows (first, last, random)
    y = torch.empty(N, dtype=torch.float64, device=DEV)
    ctx.apply(cu(x0), y)
    rows = np.concatenate([[0, N - 1, n1 - 1], rng.integers(0, N, 40)])
    ref = ro.apply_rows(x0, rows)
    got = host(y)[rows]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    # colour 0 then colour 1 of the sweep; sampled blocks checked one by one
    xg = cu(x0)
    bg = cu(b)
    ctx.sweep(bg, xg, 0, 1)
    x1 = host(xg)
    for _ in range(4):
        centre = tuple(int(D * rng.integers(0, (n1 - 1) // D + 1)) for _ in range(d))
        B, dB = ro.block_update(x0, b, centre, s)
        assert np.abs(x1[B] - (x0[B] + dB)).max() <= 1e-11 * max(np.abs(dB).max(), 1.0)
    touched = np.zeros(N, bool)
    idx = np.arange(N)
    inblk = np.ones(N, bool)
    for a in range(d):
        c = (idx // n1 ** a) % n1
        w = (s - 1) // 2
        inblk &= ((c + w) % D) <= 2 * w
    touched |= inblk
    assert np.array_equal(x1[~touched], x0[~touched])       # only colour-0 blocks changed
    ctx.sweep(bg, xg, 1, 2)
    x2 = host(xg)
    centre = (1,) + tuple(0 for _ in range(d - 1))
    B, dB = ro.block_update(x1, b, centre, s)
    assert np.abs(x2[B] - (x1[B] + dB)).max() <= 1e-11 * max(np.abs(dB).max(), 1.0)
    # a full iteration reduces the residual (property at any size)
    hist = np.zeros(3)
    ctx.iterate(bg, xg, iters=2, res_hist=hist)
    assert hist[2] < 0.9 * hist[1] < 0.9 * hist[0]


# ---- V-cycle tail in shared memory: the level spread over a cluster (DSMEM) and the CTA-local
# levels, forced at small sizes (IGA2L_VC_FORCE_CS) and at full BASELINE sizes (chosen by setup) ----
VC_SMALL = [c for c in PAR if c[6] == "vcycle"]


@pytest.mark.parametrize("cs", [2, 4, 16])
@pytest.mark.parametrize("cfg", VC_SMALL, ids=[c[0] for c in VC_SMALL])
def test_vcycle_smem_spread_level(cfg, cs, monkeypatch):
    name, d, p, q, m, s, coarse, hf = cfg
    monkeypatch.setenv("IGA2L_VC_FORCE_CS", str(cs))
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    dq = random_rhs(ctx.Nc, seed=3)
    e = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.coarse_solve(cu(dq), e)
    close(host(e), ora._csolve(dq), 1e-11)


@pytest.mark.parametrize("q,m,d", [(1, 128, 2), (1, 64, 3), (2, 512, 2)], ids=["C2", "C4", "C3"])
def test_vcycle_full_size(q, m, d):
    from oracle.multigrid import QHierarchy
    H = QHierarchy(q, m, d)
    n = H.levels[0]["n"]
    # a fine context whose aggressive second level is exactly this q-level (m_fine = 2 m)
    p = {(1, 2): 3, (1, 3): 3, (2, 2): 8}[(q, d)]
    s = 3 if p <= 4 else 7
    ctx = make_ctx(d, p, q, 2 * m, s, "vcycle", 2)
    assert ctx.Nc == n ** d
    dq = random_rhs(ctx.Nc, seed=5)
    e = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.coarse_solve(cu(dq), e)
    close(host(e), H.vcycle(dq), 1e-11)


# ---- persistent sweep (one cooperative launch per sweep, per-tile progress counters) against the
# per-colour launches: same block arithmetic, so bitwise equal; repeated launches advance the counters ----
PERSIST = [(1, 3, 48), (2, 3, 48), (3, 3, 48), (4, 3, 48), (5, 5, 48), (6, 5, 48), (7, 7, 96), (8, 7, 96)]


@pytest.mark.parametrize("p,s,m", PERSIST, ids=[f"p{c[0]}" for c in PERSIST])
def test_persistent_sweep_bitwise(p, s, m, monkeypatch):
    # the persistent kernel runs the warp-group block solve (Blk2): compare with the per-colour launches
    # of the same block solve (IGA2L_S2D_VARIANT=10), bitwise
    monkeypatch.setenv("IGA2L_S2D_VARIANT", "10")
    monkeypatch.setenv("IGA2L_SWEEP_PERSIST", "1")
    ctx = make_ctx(2, p, 1, m, s, "vcycle", 2)
    monkeypatch.setenv("IGA2L_SWEEP_PERSIST", "0")
    ref = make_ctx(2, p, 1, m, s, "vcycle", 2)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    x1, x2 = x0.clone(), x0.clone()
    for _ in range(3):
        ctx.sweep(b, x1)
        ref.sweep(b, x2)
    assert torch.equal(x1, x2)
    ctx.iterate(b, x1, iters=4)
    ref.iterate(b, x2, iters=4)
    assert torch.equal(x1, x2)


# ---- every 2D block-solve variant (DMMA default, register-blocked, warp-group) against the oracle ----
@pytest.mark.parametrize("variant", ["1", "2", "10"])
@pytest.mark.parametrize("cfg", [c for c in PAR if c[1] == 2], ids=[c[0] for c in PAR if c[1] == 2])
def test_sweep_variants_match_oracle(cfg, variant, monkeypatch):
    name, d, p, q, m, s, coarse, hf = cfg
    monkeypatch.setenv("IGA2L_S2D_VARIANT", variant)
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xg = cu(x0)
    ctx.sweep(cu(b), xg)
    close(host(xg), ora.smoother.sweep(x0.copy(), b), 1e-11)


# ---- temporal blocking (several colours per launch, halo blocks recomputed per CTA): the same block
# arithmetic as the per-colour DMMA launches, so bitwise equal; and against the oracle ----
TB_CASES = [(1, 3, 48), (2, 3, 64), (3, 3, 96), (4, 3, 64), (5, 5, 96), (6, 5, 48)]


@pytest.mark.parametrize("kc", ["2", "3"])
@pytest.mark.parametrize("p,s,m", TB_CASES, ids=[f"p{c[0]}" for c in TB_CASES])
def test_temporal_blocking_bitwise(p, s, m, kc, monkeypatch):
    monkeypatch.setenv("IGA2L_MMA_INV", "0")   # TB runs the FD GEMMs on every block
    monkeypatch.setenv("IGA2L_TB", "0")
    ref = make_ctx(2, p, 1, m, s, "vcycle", 2)
    monkeypatch.setenv("IGA2L_TB", kc)
    ctx = make_ctx(2, p, 1, m, s, "vcycle", 2)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    x1, x2 = x0.clone(), x0.clone()
    ctx.sweep(b, x1)
    monkeypatch.setenv("IGA2L_TB", "0")
    ref.sweep(b, x2)
    assert torch.equal(x1, x2)
    monkeypatch.setenv("IGA2L_TB", kc)
    ctx.sweep(b, x1, 1, 6)                 # a partial range (odd start, ragged chunk)
    monkeypatch.setenv("IGA2L_TB", "0")
    ref.sweep(b, x2, 1, 6)
    assert torch.equal(x1, x2)


# ---- 3D block-solve variants (opt-in DMMA kernel, DFMA default) against the oracle ----
@pytest.mark.parametrize("cfg", [c for c in PAR if c[1] == 3], ids=[c[0] for c in PAR if c[1] == 3])
def test_sweep3d_dmma_matches_oracle(cfg, monkeypatch):
    name, d, p, q, m, s, coarse, hf = cfg
    monkeypatch.setenv("IGA2L_S3D_MMA", "1")
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xg = cu(x0)
    ctx.sweep(cu(b), xg)
    close(host(xg), ora.smoother.sweep(x0.copy(), b), 1e-11)


# ---- exact second level at scale by Kronecker fast diagonalisation ----
EXACT_FD = [("2d_p3_exact_h", 2, 3, 1, 48, 3, "exact", 1), ("2d_p5_exact_2h", 2, 5, 1, 64, 5, "exact", 2),
            ("2d_p8_q2_exact_2h", 2, 8, 2, 40, 7, "exact", 2), ("3d_p3_exact_2h", 3, 3, 1, 16, 3, "exact", 2),
            ("3d_p5_q2_exact_h", 3, 5, 2, 10, 5, "exact", 1)]


@pytest.mark.parametrize("cfg", EXACT_FD, ids=[c[0] for c in EXACT_FD])
def test_exact_coarse_fd(cfg, monkeypatch):
    name, d, p, q, m, s, coarse, hf = cfg
    monkeypatch.setenv("IGA2L_COARSE_FD", "1")
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    ora = oracle_for(*cfg)
    dq = random_rhs(ctx.Nc, seed=4)
    e = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.coarse_solve(cu(dq), e)
    close(host(e), ora._csolve(dq), 1e-10)
    # the whole iteration with the exact second level
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    xg = cu(x0)
    ctx.iterate(cu(b), xg, iters=3)
    xo = x0.copy()
    for _ in range(3):
        ora.iterate(xo, b)
    assert np.linalg.norm(host(xg) - xo) <= 1e-10 * np.linalg.norm(xo)


def test_exact_coarse_fd_large():
    # C2-shaped problem with the exact second level at H = 2h (127^2 unknowns > the dense limit)
    ctx = make_ctx(2, 3, 1, 256, 3, "exact", 2)
    from oracle.assembly import stiffness
    A = stiffness(1, 128, 2).tocsc()
    import scipy.sparse.linalg as spla
    dq = random_rhs(ctx.Nc, seed=6)
    e = torch.empty(ctx.Nc, dtype=torch.float64, device=DEV)
    ctx.coarse_solve(cu(dq), e)
    close(host(e), spla.spsolve(A, dq), 1e-10)


@pytest.mark.parametrize("bpw", ["2", "4", "8"])
@pytest.mark.parametrize("p,s,m", [(3, 3, 96), (5, 5, 96), (8, 7, 96)], ids=["p3", "p5", "p8"])
def test_multiblock_warps_bitwise(p, s, m, bpw, monkeypatch):
    """Several blocks per warp with prefetch (IGA2L_MMA_BPW) == one block per warp, bitwise."""
    monkeypatch.setenv("IGA2L_MMA_INV", "0")   # the multi-block warps run the FD GEMMs on every block
    monkeypatch.setenv("IGA2L_MMA_BPW", "1")
    ref = make_ctx(2, p, 1, m, s, "vcycle", 2)
    ctx = make_ctx(2, p, 1, m, s, "vcycle", 2)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    x1, x2 = x0.clone(), x0.clone()
    ref.sweep(b, x1)
    monkeypatch.setenv("IGA2L_MMA_BPW", bpw)
    ctx.sweep(b, x2)
    assert torch.equal(x1, x2)


# ---- batched iterations of independent problems (fused colour launches): bitwise equal to separate calls ----
@pytest.mark.parametrize("combo", [((3, 3, 48), (4, 3, 40), (5, 5, 32)), ((2, 3, 32), (8, 7, 32)),
                                   ((3, 3, 256), (4, 3, 256), (5, 5, 256))], ids=["p345", "p28", "C2"])
def test_iterate_batch_bitwise(combo):
    ctxs, bs, xs, refs = [], [], [], []
    for i, (p, s, m) in enumerate(combo):
        st = torch.cuda.Stream(DEV)
        c = pkg.Context(2, p, 1, m, s, coarse_mode=pkg.COARSE_VCYCLE, coarse_h_factor=2, stream=st.cuda_stream)
        ctxs.append(c)
        bs.append(cu(random_rhs(c.N, seed=10 + i)))
        x0 = cu(initial_guess(c.N, seed=20 + i))
        xs.append(x0.clone())
        refs.append(x0.clone())
    torch.cuda.synchronize()
    pkg.iterate_batch(ctxs, bs, xs, iters=3)
    torch.cuda.synchronize()
    for c, b, xr in zip(ctxs, bs, refs):
        c.iterate(b, xr, iters=3)
    torch.cuda.synchronize()
    for xb, xr in zip(xs, refs):
        assert torch.equal(xb, xr)


def test_iterate_batch_fallback_mixed_dims():
    c2 = make_ctx(2, 3, 1, 48, 3, "vcycle", 2)
    c3 = make_ctx(3, 3, 1, 16, 3, "vcycle", 2)
    b2, b3 = cu(random_rhs(c2.N)), cu(random_rhs(c3.N))
    x2, x3 = cu(initial_guess(c2.N)), cu(initial_guess(c3.N))
    r2, r3 = x2.clone(), x3.clone()
    pkg.iterate_batch([c2, c3], [b2, b3], [x2, x3], iters=2)
    c2.iterate(b2, r2, iters=2)
    c3.iterate(b3, r3, iters=2)
    torch.cuda.synchronize()
    assert torch.equal(x2, r2) and torch.equal(x3, r3)


# ---- interior block inverse (s^2 <= 32: one A_B^{-1} row per lane instead of the four FD GEMMs) ----
@pytest.mark.parametrize("p,s,m", [(2, 3, 40), (3, 3, 96), (4, 3, 64), (5, 5, 96), (6, 5, 48)],
                         ids=["p2", "p3", "p4", "p5", "p6"])
def test_interior_inverse_matches_fd(p, s, m, monkeypatch):
    """IGA2L_MMA_INV=1 (opt-in) vs 0 (default): the same sweep up to rounding (both are exact block solves; the
    default path's parity with the oracle is test_one_sweep_and_phases above)."""
    monkeypatch.setenv("IGA2L_MMA_INV", "0")
    ref = make_ctx(2, p, 1, m, s, "vcycle", 2)
    ctx = make_ctx(2, p, 1, m, s, "vcycle", 2)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    x1, x2 = x0.clone(), x0.clone()
    ref.sweep(b, x1)
    monkeypatch.setenv("IGA2L_MMA_INV", "1")
    ctx.sweep(b, x2)
    scale = float(x1.abs().max())
    assert float((x1 - x2).abs().max()) <= 1e-11 * scale
    assert not torch.equal(x1, x2) or m < 4 * (p + s)   # the inverse path actually ran on interior blocks


@pytest.mark.parametrize("p,m", [(2, 24), (3, 32)], ids=["p2", "p3"])
def test_interior_inverse_3d_matches_fd(p, m, monkeypatch):
    """3D s = 3: IGA2L_S3D_INV=1 (opt-in, A_B^{-1} rows on interior blocks) vs 0 (default, shuffle FD everywhere)."""
    monkeypatch.setenv("IGA2L_S3D_INV", "0")
    ref = make_ctx(3, p, 1, m, 3, "vcycle", 2)
    ctx = make_ctx(3, p, 1, m, 3, "vcycle", 2)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    x1, x2 = x0.clone(), x0.clone()
    ref.sweep(b, x1)
    monkeypatch.setenv("IGA2L_S3D_INV", "1")
    ctx.sweep(b, x2)
    scale = float(x1.abs().max())
    assert float((x1 - x2).abs().max()) <= 1e-11 * scale
    assert not torch.equal(x1, x2)
