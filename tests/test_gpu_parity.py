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


# ---- every kernel variant a knob selects gives the oracle's result ----
@pytest.mark.parametrize("cfg", [PAR[7], PAR[8], ("3d_p5_m24", 3, 5, 2, 24, 5, "vcycle", 2)],
                         ids=["3d_p3", "3d_p5_q2", "3d_p5_m24"])
def test_3d_sweep_variants(cfg, monkeypatch):
    """3D colour kernels: v4 (CTA per block) with the window by TMA boxes and by cp.async rows
    (IGA2L_S3D_TMA=0) -- the same arithmetic in the same order, bitwise equal; v5 (warp per block, the
    default for (p, s) = (3, 3), (5, 5)) with 32-byte row loads and, on a misaligned x, 8-byte loads --
    bitwise equal to each other; all equal to the oracle's multicolour sweep (m = 24 has interior blocks)."""
    name, d, p, q, m, s, coarse, hf = cfg
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    outs = {}
    for key, env in (("v5", {"IGA2L_S3D_CHAIN": "0"}), ("v4", {"IGA2L_S3D_WARP": "0"}),
                     ("v4rows", {"IGA2L_S3D_WARP": "0", "IGA2L_S3D_TMA": "0"})):
        for k in ("IGA2L_S3D_WARP", "IGA2L_S3D_TMA", "IGA2L_S3D_CHAIN"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        xg = cu(x0)
        ctx.sweep(cu(b), xg)
        outs[key] = host(xg)
    monkeypatch.delenv("IGA2L_S3D_WARP", raising=False)
    monkeypatch.delenv("IGA2L_S3D_TMA", raising=False)
    buf = torch.zeros(ctx.N + 1, dtype=torch.float64, device=DEV)   # x at an 8-byte offset
    buf[1:] = cu(x0)
    ctx.sweep(cu(b), buf[1:])
    outs["v5mis"] = host(buf[1:])
    assert np.array_equal(outs["v4"], outs["v4rows"])
    assert np.array_equal(outs["v5"], outs["v5mis"])
    xo = x0.copy()
    if m > 20:                                   # matrix-free Kronecker oracle (pinned == TwoLevel)
        from oracle.kron import KronTwoLevel
        KronTwoLevel(d, p, q, m, s).sweep(xo, b)
    else:
        oracle_for(*cfg).smoother.sweep(xo, b)
    for key in ("v5", "v4"):
        assert np.abs(outs[key] - xo).max() <= 1e-11 * np.abs(xo).max(), key


@pytest.mark.parametrize("cfg", [PAR[2], PAR[4], PAR[5]], ids=["2d_p3", "2d_p5", "2d_p8"])
def test_2d_sweep_pdl_modes_bitwise(cfg, monkeypatch):
    """2D DMMA colour kernels with programmatic dependent launch (IGA2L_PDL = 1, 2, 3, 4: trigger at entry,
    after the window is staged, at exit, after the grid dependency wait) and without (0): the same arithmetic, bitwise equal sweeps; a
    sweep in a CUDA graph (the iteration's launch mode) equal to the eager one."""
    name, d, p, q, m, s, coarse, hf = cfg
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    outs = []
    for v in ("0", "1", "2", "3", "4"):
        monkeypatch.setenv("IGA2L_PDL", v)
        x = x0.clone()
        ctx.sweep(b, x)
        outs.append(host(x))
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
    monkeypatch.delenv("IGA2L_PDL", raising=False)
    x = x0.clone()
    ctx.sweep(b, x)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=STREAM):
        ctx.sweep(b, x)
    x.copy_(x0)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(outs[0], host(x))


@pytest.mark.parametrize("cfg", [PAR[2], PAR[3], PAR[4], PAR[5]], ids=["2d_p3", "2d_p4", "2d_p5", "2d_p8"])
def test_2d_sweep_mmg_bitwise(cfg, monkeypatch):
    """k_schwarz2d_mmg (operand fragments read per use from the interior / per-centre exports, Pab over the
    window; the default for colours larger than one wave) and k_schwarz2d_mma (fragments in registers): the
    same DMMA sequence on the same operands -> bitwise equal sweeps, equal to the oracle's sweep."""
    name, d, p, q, m, s, coarse, hf = cfg
    ctx = make_ctx(d, p, q, m, s, coarse, hf)
    b, x0 = random_rhs(ctx.N), initial_guess(ctx.N)
    outs = []
    for v in ("0", "1"):
        monkeypatch.setenv("IGA2L_MMG", v)
        x = cu(x0)
        ctx.sweep(cu(b), x)
        outs.append(host(x))
    assert np.array_equal(outs[0], outs[1])
    xo = x0.copy()
    oracle_for(*cfg).smoother.sweep(xo, b)
    assert np.abs(outs[1] - xo).max() <= 1e-11 * np.abs(xo).max()


@pytest.mark.parametrize("mb", ["0.05", "0.2"])
def test_3d_sweep_zchunk_schedule_bitwise(mb, monkeypatch):
    """The z-chunked class schedule (IGA2L_S3D_ZCHUNK_MB) reorders colours only across A-decoupled blocks of
    one last-axis class (reading A4): the swept iterate is bitwise the colour-major one."""
    ctx = make_ctx(3, 5, 2, 24, 5, "vcycle", 2)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    outs = []
    for v in ("0", mb):
        monkeypatch.setenv("IGA2L_S3D_ZCHUNK_MB", v)
        x = x0.clone()
        ctx.sweep(b, x)
        outs.append(host(x))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("p,q,m", [(3, 1, 8), (3, 1, 20), (5, 2, 10), (5, 2, 24)])
def test_3d_sweep_zchain_bitwise(p, q, m, monkeypatch):
    """The z-chain colour kernel (IGA2L_S3D_CHAIN = L: one warp sweeps ~L same-colour blocks along z, each plane
    group's pass x / y shared by the two blocks whose windows hold it) performs v5's arithmetic per point in
    the same order: bitwise equal sweeps for every segment length, incl. segments longer than the column and
    the misaligned-x fallback; and equal to the oracle's sweep."""
    ctx = make_ctx(3, p, q, m, p, "vcycle", 2)
    b, x0 = cu(random_rhs(ctx.N)), cu(initial_guess(ctx.N))
    outs = {}
    for L in ("0", "1", "2", "3", "64", "auto"):
        if L == "auto":
            monkeypatch.delenv("IGA2L_S3D_CHAIN", raising=False)     # the default (chain at p = 5, v5 at p = 3)
        else:
            monkeypatch.setenv("IGA2L_S3D_CHAIN", L)
        x = x0.clone()
        ctx.sweep(b, x)
        outs[L] = host(x)
    monkeypatch.setenv("IGA2L_S3D_CHAIN", "2")
    for lv in ("1", "4"):                        # row-load width A/B knob
        monkeypatch.setenv("IGA2L_S3D_CHAIN_LV", lv)
        x = x0.clone()
        ctx.sweep(b, x)
        outs["lv" + lv] = host(x)
    monkeypatch.delenv("IGA2L_S3D_CHAIN_LV", raising=False)
    for nw in ("4", "1"):                        # warps per CTA A/B knob (default 2)
        monkeypatch.setenv("IGA2L_S3D_NW", nw)
        x = x0.clone()
        ctx.sweep(b, x)
        outs["nw" + nw] = host(x)
    monkeypatch.delenv("IGA2L_S3D_NW", raising=False)
    buf = torch.zeros(ctx.N + 1, dtype=torch.float64, device=DEV)   # x at an 8-byte offset: v5's fallback
    buf[1:] = x0
    ctx.sweep(b, buf[1:])
    outs["mis"] = host(buf[1:])
    for L, o in outs.items():
        assert np.array_equal(outs["0"], o), L
    xo = host(x0)
    if m > 20:                                   # matrix-free Kronecker oracle (pinned == TwoLevel)
        from oracle.kron import KronTwoLevel
        KronTwoLevel(3, p, q, m, p).sweep(xo, host(b))
    else:
        oracle_for(f"3d_p{p}", 3, p, q, m, p, "vcycle", 2).smoother.sweep(xo, host(b))
    assert np.abs(outs["2"] - xo).max() <= 1e-11 * np.abs(xo).max()


@pytest.mark.parametrize("p,m", [(3, 20), (5, 12)])
@pytest.mark.parametrize("env", [{"IGA2L_APPLY_STREAM": "0"}, {"IGA2L_STREAM_CFG": "1"}, {"IGA2L_STREAM_CFG": "2"},
                                 {"IGA2L_STREAM_CFG": "3"}, {"IGA2L_STREAM_CFG": "4"}, {"IGA2L_STREAM_CFG": "5"}],
                         ids=["tiled", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_3d_apply_variants(p, m, env, monkeypatch):
    """3D residual: the tiled kernel and every streaming configuration against the assembled operator,
    and the residual norm over exactly the partials each variant writes."""
    from oracle.assembly import stiffness
    ctx = make_ctx(3, p, 1, m, 3 if p <= 4 else 5, "vcycle", 2)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    x, b = initial_guess(ctx.N, seed=2), random_rhs(ctx.N, seed=3)
    y = torch.empty(ctx.N, dtype=torch.float64, device=DEV)
    ctx.apply(cu(x), y)
    ref = stiffness(p, m, 3) @ x
    assert np.abs(host(y) - ref).max() <= 1e-13 * np.abs(ref).max()
    rn = ctx.residual_norm(cu(b), cu(x))
    assert abs(rn - np.linalg.norm(b - ref)) <= 1e-12 * np.linalg.norm(b - ref)


@pytest.mark.parametrize("p", [1, 2, 4, 6, 7, 8])
@pytest.mark.parametrize("m", [9, 37])
def test_3d_apply_every_degree(p, m):
    """The streaming 3D residual kernel is instantiated for p = 1..8 (the q-level residuals use p = 1, 2): every
    degree the configs do not exercise against the oracle's Kronecker operator, one tile (m = 9) and several
    tiles with ragged tails in x, y and the z segments (m = 37)."""
    from oracle.kron import KronOperator
    ctx = make_ctx(3, p, 1, m, 3 if p <= 4 else (5 if p <= 6 else 7), "exact", 1)
    x, b = initial_guess(ctx.N, seed=4), random_rhs(ctx.N, seed=5)
    y = torch.empty(ctx.N, dtype=torch.float64, device=DEV)
    ctx.apply(cu(x), y)
    ref = KronOperator(p, m, 3).apply(x)
    assert np.abs(host(y) - ref).max() <= 1e-13 * np.abs(ref).max()
    rn = ctx.residual_norm(cu(b), cu(x))
    assert abs(rn - np.linalg.norm(b - ref)) <= 1e-12 * np.linalg.norm(b - ref)

