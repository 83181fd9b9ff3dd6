"""Pins for oracle/bspline.py against what the paper and mathematics fix (not against itself)."""
import math

import numpy as np
import pytest
import scipy.interpolate as si

from oracle.bspline import basis, basis_deriv, knot_vector

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")


def test_knot_vector_example():
    # ξ_1..ξ_{p+1} = 0, ξ_{p+i+1} = i/m, ξ_{p+m+1}.. = 1; SPEC S:61 example (p=2, m=4)
    assert np.array_equal(knot_vector(2, 4), [0, 0, 0, 0.25, 0.5, 0.75, 1, 1, 1])
    assert np.array_equal(knot_vector(1, 2), [0, 0, 0.5, 1, 1])
    assert len(knot_vector(3, 8)) == 2 * 3 + 8 + 1


@pytest.mark.parametrize("p", range(0, 9))
def test_partition_nonneg_support_dimension(p):
    m = 7
    xi = knot_vector(p, m)
    xs = np.concatenate([np.random.default_rng(p).uniform(0, 1, 200), [0.0, 1.0, 3 / 7]])
    N = basis(xi, p, xs)
    assert N.shape[1] == m + p                      # full dimension; Dirichlet keeps m+p-2
    assert np.allclose(N.sum(axis=1), 1.0, atol=1e-12, rtol=0)
    assert (N >= -1e-15).all()
    for i in range(m + p):                          # support of N_i^p is [ξ_i, ξ_{i+p+1}]
        out = (xs < xi[i]) | (xs > xi[i + p + 1])
        assert np.all(N[out, i] == 0.0)


@pytest.mark.parametrize("p", range(1, 9))
def test_matches_scipy_bspline(p):
    # independent library implementation of B-spline evaluation (de Boor in scipy)
    m = 6
    xi = knot_vector(p, m)
    xs = np.random.default_rng(10 + p).uniform(0, 1, 50)
    N = basis(xi, p, xs)
    for i in range(m + p):
        c = np.zeros(m + p)
        c[i] = 1.0
        ref = si.BSpline(xi, c, p, extrapolate=False)(xs)
        assert np.allclose(N[:, i], ref, atol=1e-13, rtol=0)


def cardinal(n, t):
    """Cardinal B-spline of degree n on [0, n+1] by the truncated-power closed form
    N_n(t) = 1/n! Σ_{k=0}^{n+1} (-1)^k C(n+1,k) (t-k)_+^n (textbook identity)."""
    t = np.asarray(t, dtype=float)
    return sum((-1) ** k * math.comb(n + 1, k) * np.maximum(t - k, 0.0) ** n
               for k in range(n + 2)) / math.factorial(n)


@pytest.mark.parametrize("p", range(1, 9))
def test_interior_function_is_translated_cardinal_bspline(p):
    m = 3 * p + 4
    h = 1.0 / m
    xi = knot_vector(p, m)
    xs = np.random.default_rng(p).uniform(0, 1, 300)
    N = basis(xi, p, xs)
    for i in range(p, m):                           # full 0-based index i: knots i..i+p+1 all simple
        t = (xs - xi[i]) / h
        ref = np.where((t >= 0) & (t <= p + 1), cardinal(p, t), 0.0)   # formula cancels to ~1e-11 outside
        assert np.allclose(N[:, i], ref, atol=1e-10, rtol=0)


@pytest.mark.parametrize("p", range(1, 9))
def test_first_function_is_bernstein(p):
    # open knots: N_1^p(x) = (1 - x/h)^p on [0, h]
    m = 5
    xs = np.linspace(0, 1 / m, 17)
    N = basis(knot_vector(p, m), p, xs)
    assert np.allclose(N[:, 0], (1 - xs * m) ** p, atol=1e-13)


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
def test_derivative_finite_difference_and_sum(p):
    m = 5
    xi = knot_vector(p, m)
    xs = np.random.default_rng(3).uniform(0.01, 0.99, 40)
    xs = xs[np.min(np.abs(xs[:, None] - np.arange(m + 1)[None, :] / m), axis=1) > 1e-4]
    dN = basis_deriv(xi, p, xs)
    eps = 1e-6
    fd = (basis(xi, p, xs + eps) - basis(xi, p, xs - eps)) / (2 * eps)
    assert np.allclose(dN, fd, atol=1e-5 * m * p, rtol=1e-6)
    assert np.allclose(dN.sum(axis=1), 0.0, atol=1e-10)


@pytest.mark.parametrize("p,m", [(1, 3), (2, 5), (3, 7), (5, 9), (8, 12)])
def test_span_basis_is_bitwise_the_global_recursion(p, m):
    """span_basis (the p+1 functions alive on one span, from the knot window) == the columns of the
    full Cox-de Boor evaluation, bitwise, on every span incl. the repeated end knots."""
    from oracle.bspline import basis, basis_deriv, knot_vector, span_basis, span_rule
    xi = knot_vector(p, m)
    for e in range(m):
        xs, _ = span_rule(m, e, p + 3)
        assert np.array_equal(span_basis(xi, p, e, xs), basis(xi, p, xs)[:, e:e + p + 1])
        assert np.array_equal(span_basis(xi, p, e, xs, deriv=True), basis_deriv(xi, p, xs)[:, e:e + p + 1])
