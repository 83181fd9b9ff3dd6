"""Pins for oracle/twolevel.py (Algorithm 1): fixed points, convergence to the direct
solution, the dense error operator vs the measured factor, and the paper's measured / LFA
factors (Tables 1-3) for the lexicographic Schwarz order within 0.05."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle.twolevel import TwoLevel, paper_block_size
from synthetic_inputs import initial_guess, random_rhs


def test_paper_block_sizes():
    # P:312 / P:406
    assert [paper_block_size(p) for p in range(2, 9)] == [3, 3, 3, 5, 5, 7, 7]


def test_hierarchy_sizes():
    # S:365-366 examples: coarse (1+16-2)^2 = 225 at h, (1+8-2)^2 = 49 at 2h
    assert TwoLevel(2, 2, 1, 16, coarse="exact", h_factor=1).R.shape[0] == 225
    assert TwoLevel(2, 3, 1, 16, coarse="exact", h_factor=2).R.shape[0] == 49
    assert [lv["m"] for lv in TwoLevel(2, 3, 1, 64, coarse="vcycle", h_factor=2).mg.levels] == [32, 16, 8]


@pytest.mark.parametrize("kw", [dict(coarse="exact", h_factor=1), dict(coarse="vcycle", h_factor=2)])
def test_zero_stays_zero_and_solution_is_fixed_point(kw):
    tl = TwoLevel(2, 3, 1, 16, **kw)
    x = np.zeros(tl.N)
    tl.iterate(x, np.zeros(tl.N))
    assert not np.any(x)
    b = random_rhs(tl.N)
    u = spla.spsolve(tl.A.tocsc(), b)
    x = u.copy()
    tl.iterate(x, b)
    assert np.linalg.norm(b - tl.A @ x) <= 1e-12 * np.linalg.norm(b)


@pytest.mark.parametrize("d,p,q,m,kw", [(2, 3, 1, 16, dict(coarse="vcycle", h_factor=2)),
                                        (2, 5, 2, 16, dict(coarse="exact", h_factor=1)),
                                        (3, 3, 1, 8, dict(coarse="vcycle", h_factor=2))])
def test_converges_to_direct_solution(d, p, q, m, kw):
    tl = TwoLevel(d, p, q, m, **kw)
    b = random_rhs(tl.N)
    u = spla.spsolve(tl.A.tocsc(), b)
    x, it, hist = tl.solve(b, initial_guess(tl.N), rtol=1e-12, maxit=60)
    assert hist[-1] <= 1e-12 * hist[0]
    assert np.linalg.norm(x - u) <= 1e-9 * np.linalg.norm(u)


def test_c1_error_operator_spectral_radius_matches_measured_factor():
    # C1 (BASELINE configs[0]): the dense error operator E pins the "conv. factor" metric;
    # its spectral radius must agree with the measured asymptotic factor within 2%.
    tl = TwoLevel(2, 2, 1, 16, coarse="exact", h_factor=1)
    E = tl.error_operator()
    rho = np.abs(np.linalg.eigvals(E)).max()
    rate, _ = tl.rate(initial_guess(tl.N), iters=40)
    assert abs(rate - rho) <= 0.02 * rho, (rate, rho)
    assert rho < 0.1216        # better than the paper's lex ρ_h for p=2, 9p


# Table 1 (same h, exact coarse, q = 1): ρ_h column, lex order, m = 64.
@pytest.mark.parametrize("p,s,paper,iters", [(3, 3, 0.2141, 25), (4, 3, 0.4558, 25), (6, 5, 0.4555, 40)])
def test_table1_measured_factor(p, s, paper, iters):
    tl = TwoLevel(2, p, 1, 64, s=s, coarse="exact", h_factor=1, order="lex")
    rate, _ = tl.rate(initial_guess(tl.N), iters=iters)
    assert abs(rate - paper) <= 0.05, rate


def test_table2_vcycle_factor():
    # Table 2: p = 4, 9p, one V(1,1) at the same h: ρ_3g = 0.4566
    tl = TwoLevel(2, 4, 1, 64, s=3, coarse="vcycle", h_factor=1, order="lex")
    rate, _ = tl.rate(initial_guess(tl.N), iters=25)
    assert abs(rate - 0.4566) <= 0.05, rate


def test_table3_aggressive_factor():
    # Table 3: p = 4, 9p, exact q-level at H = 2h: ρ_2g^ag = 0.4566
    tl = TwoLevel(2, 4, 1, 64, s=3, coarse="exact", h_factor=2, order="lex")
    rate, _ = tl.rate(initial_guess(tl.N), iters=25)
    assert abs(rate - 0.4566) <= 0.05, rate
