"""Pins for oracle/assembly.py: closed forms, exact symbolic integrals, FE special cases,
structural invariants and the O(h^{p+1}) convergence order."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import assembly as A

GOLD = os.path.join(os.path.dirname(__file__), "golden", "bspline_boundary_rows.json")


def cardinal(n, t, deriv=0):
    """Cardinal B-spline of degree n (or its deriv-th derivative) at an INTEGER t, exactly, by the
    truncated-power closed form N_n(t) = 1/n! Σ_{k=0}^{n+1} (-1)^k C(n+1,k) (t-k)_+^n."""
    e = n - deriv
    c = math.factorial(n) // math.factorial(e)
    s = sum(Fraction((-1) ** k * math.comb(n + 1, k) * c * (t - k) ** e)
            for k in range(n + 2) if t - k > 0)
    return float(s / math.factorial(n))


def test_p1_fe_rows():
    # linear FE: K rows (-1, 2, -1)/h, M rows h(1, 4, 1)/6
    m = 8
    h = 1 / m
    K, M = A.matrices_1d(1, m)
    for i in range(1, K.shape[0] - 1):
        assert np.allclose(K[i, i - 1:i + 2] * h, [-1, 2, -1], atol=1e-13)
        assert np.allclose(M[i, i - 1:i + 2] / h, [1 / 6, 4 / 6, 1 / 6], atol=1e-14)


@pytest.mark.parametrize("p", range(1, 9))
def test_interior_rows_cardinal_closed_form(p):
    # M_{i,i+t} = h N_{2p+1}(p+1+t), K_{i,i+t} = -h^{-1} N''_{2p+1}(p+1+t) (autocorrelation of
    # cardinal B-splines; e.g. p=2: M/h = [1,26,66,26,1]/120, K h = [-1,-2,6,-2,-1]/6)
    m = 4 * p + 6
    h = 1 / m
    K, M = A.matrices_1d(p, m)
    i = K.shape[0] // 2
    for t in range(-p, p + 1):
        assert abs(M[i, i + t] / h - cardinal(2 * p + 1, p + 1 + t)) < 1e-13
        assert abs(K[i, i + t] * h + cardinal(2 * p + 1, p + 1 + t, deriv=2)) < 1e-11
    if p == 2:
        assert np.allclose(M[i, i - 2:i + 3] / h, np.array([1, 26, 66, 26, 1]) / 120, atol=1e-14)
        assert np.allclose(K[i, i - 2:i + 3] * h, np.array([-1, -2, 6, -2, -1]) / 6, atol=1e-13)


def _sympy_rows(p, m, nrows):
    sympy = pytest.importorskip("sympy")
    x = sympy.Symbol("x")
    kn = [sympy.Integer(0)] * (p + 1) + [sympy.Rational(i, m) for i in range(1, m)] + [sympy.Integer(1)] * (p + 1)
    B = sympy.bspline_basis_set(p, kn, x)[1:-1]                       # constrained basis
    Kh, Mh = [], []
    for i in range(nrows):
        Kh.append([sympy.integrate(sympy.diff(B[i], x) * sympy.diff(B[j], x), (x, 0, 1)) / m
                   for j in range(len(B))])
        Mh.append([sympy.integrate(B[i] * B[j], (x, 0, 1)) * m for j in range(len(B))])
    return Kh, Mh


@pytest.mark.parametrize("key,p,m,nrows", [("p2_m5", 2, 5, 3), ("p3_m7", 3, 7, 2)])
def test_boundary_rows_exact_rationals(key, p, m, nrows):
    gold = json.load(open(GOLD))[key]
    Kh, Mh = _sympy_rows(p, m, nrows)
    K, M = A.matrices_1d(p, m)
    for i in range(nrows):
        gk = [Fraction(s) for s in gold["K_times_h"][i]]
        gm = [Fraction(s) for s in gold["M_over_h"][i]]
        lo = max(0, i - p)
        # golden strings agree with exact symbolic integration ...
        assert [Fraction(str(v)) for v in Kh[i][lo:lo + len(gk)]] == gk
        assert [Fraction(str(v)) for v in Mh[i][lo:lo + len(gm)]] == gm
        # ... and the oracle's quadrature reproduces the exact rows to rounding
        assert np.allclose(K[i] / m, [float(v) for v in Kh[i]], atol=2e-15, rtol=0)
        assert np.allclose(M[i] * m, [float(v) for v in Mh[i]], atol=2e-15, rtol=0)


@pytest.mark.parametrize("d,p,m", [(2, 1, 6), (2, 3, 7), (2, 5, 6), (3, 2, 4), (3, 3, 3)])
def test_elementwise_equals_kronecker_and_structure(d, p, m):
    Ae = A.stiffness_elementwise(p, m, d)
    Ak = A.stiffness_kron(p, m, d)
    assert abs(Ae - Ak).max() < 1e-13 * abs(Ae).max()
    assert abs(Ae - Ae.T).max() < 1e-12                            # symmetric
    ev = np.linalg.eigvalsh(Ae.toarray())
    assert ev.min() > 0                                            # SPD (coercivity)
    # Neumann operator annihilates constants
    An = A.stiffness_elementwise(p, m, d, constrained=False)
    assert np.abs(An @ np.ones(An.shape[0])).max() < 1e-11
    # nnz per interior row = (2p+1)^d stencil
    assert Ae.getnnz(axis=1).max() == min(2 * p + 1, m + p - 2) ** d


def test_p1_2d_stencil():
    # bilinear FE: (1/3)[-1 -1 -1; -1 8 -1; -1 -1 -1]
    m = 6
    Aq = A.stiffness(1, m, 2).toarray()
    n = m - 1
    c = 2 + n * 2
    row = Aq[c].reshape(n, n)
    assert np.allclose(row[1:4, 1:4] * 3, [[-1, -1, -1], [-1, 8, -1], [-1, -1, -1]], atol=1e-13)


@pytest.mark.parametrize("d,p,m", [(2, 2, 5), (3, 3, 3)])
def test_load_separable_equals_elementwise(d, p, m):
    assert np.allclose(A.load_sine(p, m, d), A.load_sine_elementwise(p, m, d), atol=1e-14, rtol=1e-13)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_l2_convergence_order(p):
    # O(h^{p+1}) for u = sin(pi x) sin(pi y): observed order >= p + 0.9 from m=8 to 16
    errs = []
    for m in (8, 16):
        Ap = A.stiffness(p, m, 2).tocsc()
        u = spla.spsolve(Ap, A.load_sine(p, m, 2))
        errs.append(A.l2_error_sine(p, m, 2, u))
    order = np.log2(errs[0] / errs[1])
    assert order >= p + 0.9, (errs, order)
