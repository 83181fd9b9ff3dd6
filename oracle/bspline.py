"""ORACLE (test infrastructure only) — univariate B-splines, straight from P:90-113.

Indices: the paper numbers knots ξ_1..ξ_{2p+m+1} and basis functions
N_1..N_{m+p} from 1.  Here arrays are 0-based, so paper index ``i`` is
array index ``i-1``.  The Dirichlet space S_h^p keeps N_2..N_{p+m-1}
(P:98), i.e. full 0-based indices 1..m+p-2.
"""
import numpy as np


def knot_vector(p, m):
    """Uniform open knot vector Ξ_{p,h}.

    ξ_1 = … = ξ_{p+1} = 0, ξ_{p+i+1} = i/m for i = 0..m, ξ_{p+m+1} = … = ξ_{2p+m+1} = 1.
    """
    if p < 0 or m < 1:
        raise ValueError("need p >= 0, m >= 1")
    xi = np.empty(2 * p + m + 1)
    xi[: p + 1] = 0.0
    for i in range(m + 1):
        xi[p + i] = i / m          # paper ξ_{p+i+1}  ->  0-based p+i
    xi[p + m:] = 1.0
    return xi


def _degree0(xi, xs):
    """N_i^0: 1 on [ξ_i, ξ_{i+1}), 0 otherwise.

    Convention (A18): the last non-empty span is closed at ξ = 1 so
    the basis covers [0, 1].
    """
    n0 = len(xi) - 1
    N = np.zeros((len(xs), n0))
    for i in range(n0):
        N[:, i] = ((xs >= xi[i]) & (xs < xi[i + 1])).astype(float)
    last = max(i for i in range(n0) if xi[i] < xi[i + 1])
    N[xs == xi[-1], last] = 1.0
    return N


def basis(xi, k, xs):
    """All N_i^k(ξ) for i = 1..len(xi)-k-1 by the Cox–de Boor recursion.

    N_i^k = (ξ-ξ_i)/(ξ_{i+k}-ξ_i) N_i^{k-1} + (ξ_{i+k+1}-ξ)/(ξ_{i+k+1}-ξ_{i+1}) N_{i+1}^{k-1},
    with fractions 0/0 taken as zero.  Returns an array [len(xs), n_funcs].
    """
    xs = np.atleast_1d(np.asarray(xs, dtype=float))
    N = _degree0(xi, xs)
    for kk in range(1, k + 1):
        nk = N.shape[1] - 1
        Nn = np.zeros((len(xs), nk))
        for i in range(nk):
            d1 = xi[i + kk] - xi[i]
            d2 = xi[i + kk + 1] - xi[i + 1]
            t1 = (xs - xi[i]) / d1 * N[:, i] if d1 != 0.0 else 0.0
            t2 = (xi[i + kk + 1] - xs) / d2 * N[:, i + 1] if d2 != 0.0 else 0.0
            Nn[:, i] = t1 + t2
        N = Nn
    return N


def span_basis(xi, k, e, xs, deriv=False):
    """The k+1 functions N_e^k .. N_{e+k}^k (0-based, full numbering) that can be non-zero on the
    knot span [ξ_{e+k}, ξ_{e+k+1}), at points xs inside that span.  They depend only on the knots
    ξ_e .. ξ_{e+2k+1}, so this is ``basis(xi, k, xs)[:, e:e+k+1]`` (or ``basis_deriv``) computed by
    the same recursion on that knot window: the same operations on the same values, i.e. bitwise
    equal (pinned in tests/test_oracle_bspline.py), without the functions that vanish there."""
    sub = xi[e:e + 2 * k + 2]
    return basis_deriv(sub, k, xs) if deriv else basis(sub, k, xs)


def basis_deriv(xi, k, xs):
    """d/dξ N_i^k by the standard degree-reduction rule (needed by a(u,v)):

    N_i^k' = k/(ξ_{i+k}-ξ_i) N_i^{k-1} - k/(ξ_{i+k+1}-ξ_{i+1}) N_{i+1}^{k-1}, 0/0 := 0.
    """
    xs = np.atleast_1d(np.asarray(xs, dtype=float))
    Nl = basis(xi, k - 1, xs)
    nk = Nl.shape[1] - 1
    dN = np.zeros((len(xs), nk))
    for i in range(nk):
        d1 = xi[i + k] - xi[i]
        d2 = xi[i + k + 1] - xi[i + 1]
        t1 = k / d1 * Nl[:, i] if d1 != 0.0 else 0.0
        t2 = k / d2 * Nl[:, i + 1] if d2 != 0.0 else 0.0
        dN[:, i] = t1 - t2
    return dN


def gauss_rule(n, a, b):
    """n-point Gauss–Legendre rule on [a, b] (library primitive: numpy leggauss)."""
    g, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (a + b) + 0.5 * (b - a) * g, 0.5 * (b - a) * w


def span_rule(m, e, n):
    """Gauss rule on knot span I_{e+1} = (e h, (e+1) h), h = 1/m."""
    return gauss_rule(n, e / m, (e + 1) / m)
