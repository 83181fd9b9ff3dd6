"""Pins for oracle/transfer.py: exact symbolic cross-mass integrals, the lumping closed form,
constant preservation, knot-insertion columns, nestedness (independent scipy evaluation) and the
Galerkin identity A_{2h} = P^T A_h P for nested spaces."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.interpolate as si

from oracle import assembly as A
from oracle import transfer as T
from oracle.bspline import knot_vector

GOLD = os.path.join(os.path.dirname(__file__), "golden", "bspline_boundary_rows.json")


@pytest.mark.parametrize("q,m", [(1, 6), (2, 7), (2, 16)])
def test_lumped_mass_closed_form(q, m):
    # ∫ N_i^q = (ξ_{i+q+1} - ξ_i)/(q+1) (textbook); constrained rows are full indices 1..m+q-2
    xi = knot_vector(q, m)
    D = T.lumped_mass_1d(q, m)
    ref = np.array([(xi[i + q + 1] - xi[i]) / (q + 1) for i in range(1, m + q - 1)])
    assert np.allclose(D, ref, atol=1e-15, rtol=1e-14)


@pytest.mark.parametrize("p,q,m", [(2, 1, 6), (3, 1, 7), (4, 2, 7)])
def test_cross_mass_exact(p, q, m):
    sympy = pytest.importorskip("sympy")
    x = sympy.Symbol("x")

    def kn(k):
        return [sympy.Integer(0)] * (k + 1) + [sympy.Rational(i, m) for i in range(1, m)] + [sympy.Integer(1)] * (k + 1)

    Bq = sympy.bspline_basis_set(q, kn(q), x)[1:-1]
    Bp = sympy.bspline_basis_set(p, kn(p), x)[1:-1]
    Mc = A.cross_mass_1d(q, p, m)
    for i in (0, 1, len(Bq) // 2, len(Bq) - 1):
        exact = [float(sympy.integrate(Bq[i] * Bp[j], (x, 0, 1))) for j in range(len(Bp))]
        assert np.allclose(Mc[i], exact, atol=2e-16, rtol=1e-14)


def test_cross_mass_interior_cardinal():
    # interior rows of M_c/h are cardinal values of degree p+q+1: (2,1) [1,11,11,1]/24, (3,1) [1,26,66,26,1]/120
    for (p, q, ref) in [(2, 1, np.array([1, 11, 11, 1]) / 24), (3, 1, np.array([1, 26, 66, 26, 1]) / 120)]:
        m = 20
        Mc = A.cross_mass_1d(q, p, m) * m
        row = Mc[m // 2]
        nz = row[np.abs(row) > 1e-14]
        assert np.allclose(nz, ref, atol=1e-14)


def test_restriction_row_golden_and_constants():
    gold = json.load(open(GOLD))["p3_m7"]["R1_row0_p3_q1"]
    R1 = T.degree_restriction_1d(3, 1, 7)
    assert np.allclose(R1[0, :4], [float(Fraction(s)) for s in gold], atol=1e-15)
    assert np.all(R1[0, 4:] == 0)
    # D/h = 1 for every constrained q=1 function
    assert np.allclose(T.lumped_mass_1d(1, 7) * 7, 1.0)
    # unconstrained restriction preserves constants: D_full^{-1} M_c,full 1 = 1
    for p, q, m in [(3, 1, 9), (5, 2, 8), (8, 2, 12)]:
        _, Mq = A.matrices_1d(q, m, constrained=False)
        Mc = A.cross_mass_1d(q, p, m, constrained=False)
        R = Mc / Mq.sum(axis=1)[:, None]
        assert np.allclose(R @ np.ones(m + p), 1.0, atol=1e-14)


def test_knot_insertion_columns():
    # q=1 interior column (1/2, 1, 1/2); q=2 interior column (1/4, 3/4, 3/4, 1/4)
    P1 = T.mesh_prolongation_1d(1, 8)
    col = P1[:, 3]
    assert np.allclose(col[np.abs(col) > 0], [0.5, 1, 0.5], atol=1e-14)
    P2 = T.mesh_prolongation_1d(2, 8)
    col = P2[:, 4]
    assert np.allclose(col[np.abs(col) > 0], [0.25, 0.75, 0.75, 0.25], atol=1e-14)


@pytest.mark.parametrize("q,mc", [(1, 4), (2, 5), (2, 8), (3, 4)])
def test_nestedness_scipy(q, mc):
    # the spline with coefficients P c equals the coarse spline pointwise (independent evaluator)
    P = T.mesh_prolongation_1d(q, mc, constrained=False)
    c = np.random.default_rng(q * 10 + mc).uniform(-1, 1, mc + q)
    xs = np.random.default_rng(1).uniform(0, 1, 100)
    coarse = si.BSpline(knot_vector(q, mc), c, q)(xs)
    fine = si.BSpline(knot_vector(q, 2 * mc), P @ c, q)(xs)
    assert np.allclose(coarse, fine, atol=1e-12)


@pytest.mark.parametrize("q,mc,d", [(1, 4, 2), (2, 4, 2), (1, 3, 3)])
def test_galerkin_identity(q, mc, d):
    P = T.mesh_prolongation(q, mc, d)
    Ah = A.stiffness(q, 2 * mc, d)
    A2h = A.stiffness(q, mc, d)
    G = (P.T @ Ah @ P).toarray()
    assert np.abs(G - A2h.toarray()).max() < 1e-13 * np.abs(A2h.toarray()).max()


def test_aggressive_sizes():
    p, q, m, d = 3, 1, 16, 2
    R = T.restriction(p, q, m, d, 2)
    assert R.shape == ((q + m // 2 - 2) ** d, (p + m - 2) ** d)
    R1 = T.restriction(p, q, m, d, 1)
    assert R1.shape == ((q + m - 2) ** d, (p + m - 2) ** d)
