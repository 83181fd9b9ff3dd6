"""Pins of the quarter-annulus NURBS oracle (oracle/annulus.py):
exact geometry, NURBS partition of unity, SPD stiffness, the manufactured solution's L2 convergence order,
the tensor structure of the operator on this map, the exact nested embedding, and a converging two-level
iteration.  Table 5's iteration counts are context only (the paper's three-colour order, reading A4/A21)."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import annulus as an
from oracle.bspline import knot_vector, span_basis


def test_geometry_is_the_quarter_annulus():
    xi = np.linspace(0.0, 1.0, 11)
    for eta, rad in ((0.0, an.R_IN), (1.0, an.R_OUT)):
        X, _ = an.geometry(xi, np.full_like(xi, eta))
        assert np.abs(np.hypot(X[:, 0], X[:, 1]) - rad).max() < 1e-15
    X0, _ = an.geometry(np.zeros(5), np.linspace(0, 1, 5))
    X1, _ = an.geometry(np.ones(5), np.linspace(0, 1, 5))
    assert np.abs(X0[:, 1]).max() < 1e-16 and np.abs(X1[:, 0]).max() < 1e-16
    # area = ∫ |det J| = π (R² - r²) / 4, and the Jacobian columns are orthogonal (F = ρ(η) c(ξ), |c| = 1)
    from oracle.bspline import gauss_rule
    g, w = (np.asarray(v) for v in gauss_rule(12, 0.0, 1.0))
    XI, ETA = np.meshgrid(g, g)
    _, J = an.geometry(XI.ravel(), ETA.ravel())
    det = np.abs(J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0])
    area = (w[:, None] * w[None, :]).ravel() @ det
    assert abs(area - np.pi * (an.R_OUT ** 2 - an.R_IN ** 2) / 4) < 1e-12
    assert np.abs(np.einsum("kij,ki->k", J[:, :, :1], J[:, :, 1])).max() < 1e-14


@pytest.mark.parametrize("p,m", [(2, 4), (3, 8), (5, 6)])
def test_nurbs_partition_of_unity_and_weight_function(p, m):
    xs = np.linspace(0.01, 0.99, 37)
    kv = knot_vector(p, m)
    w = an.nurbs_weights(p, m)
    for e in range(m):
        sel = xs[(xs >= e / m) & (xs < (e + 1) / m)]
        if not len(sel):
            continue
        R, _ = an.nurbs_1d(p, m, sel, e)
        assert np.abs(R.sum(axis=1) - 1).max() < 1e-14
        Wref, _ = an.arc_weight(sel)                             # W is exactly in the refined space
        assert np.abs(span_basis(kv, p, e, sel) @ w[e:e + p + 1] - Wref).max() < 1e-14


@pytest.mark.parametrize("p", [3, 4])
def test_stiffness_spd_and_l2_convergence(p):
    errs = []
    for m in (8, 16):
        g = an.assemble(p, m, want=("A", "b"))
        A = g["A"]
        assert abs(A - A.T).max() < 1e-13
        if m == 8:
            assert np.linalg.eigvalsh(A.toarray()).min() > 0
        errs.append(an.l2_error(p, m, spla.spsolve(A.tocsc(), g["b"])))
    assert np.log2(errs[0] / errs[1]) > p + 0.8, errs      # O(h^{p+1})


@pytest.mark.parametrize("p,m", [(3, 6), (5, 8)])
def test_tensor_structure_on_the_map(p, m):
    """The GPU path applies A = My ⊗ Kx + Ky ⊗ Mx (per-axis 1D tables): equal to the 2D element assembly."""
    A = an.assemble(p, m)["A"].toarray()
    Kx, Mx, Ky, My = an.separable_1d(p, m)
    assert np.abs(np.kron(My, Kx) + np.kron(Ky, Mx) - A).max() < 1e-13 * np.abs(A).max()


def test_embedding_is_exact():
    """P maps the coarse coefficients of a degree-q NURBS function on mc spans to the fine coefficients
    of the SAME function on 2 mc spans (nested spaces, reading A8): compare point values."""
    q, mc = 2, 4
    P = an.embedding(q, mc).toarray()
    rng = np.random.default_rng(0)
    cc = rng.uniform(-1, 1, (mc + q - 2) ** 2)
    cf = P @ cc

    def values(c, m, pts):
        n1 = m + q - 2
        C = np.zeros((n1 + 2, n1 + 2))
        C[1:-1, 1:-1] = c.reshape(n1, n1)
        out = []
        for x, y in pts:
            ex, ey = min(int(x * m), m - 1), min(int(y * m), m - 1)
            R, _ = an.nurbs_1d(q, m, np.array([x]), ex)
            N = span_basis(knot_vector(q, m), q, ey, np.array([y]))
            out.append(float(N[0] @ C[ey:ey + q + 1, ex:ex + q + 1] @ R[0]))
        return np.array(out)
    pts = rng.uniform(0, 1, (20, 2))
    assert np.abs(values(cf, 2 * mc, pts) - values(cc, mc, pts)).max() < 1e-13


@pytest.mark.parametrize("coarse", ["vcycle", "exact"])
def test_two_level_converges_to_direct_solution(coarse):
    tl = an.AnnulusTwoLevel(3, 16, 3, coarse=coarse)
    u = spla.spsolve(tl.A.tocsc(), tl.b)
    x, it, rr = tl.solve(tl.b, np.random.default_rng(0).uniform(-1, 1, tl.N), rtol=1e-8)
    assert rr <= 1e-8 and it <= 15
    x, it, rr = tl.solve(tl.b, x, rtol=1e-4)                   # to ~1e-12 of the initial residual overall
    assert np.linalg.norm(x - u) <= 1e-7 * np.linalg.norm(u)
    y = u.copy()
    tl.iterate(y, tl.b)                                       # the solution is a fixed point
    assert np.linalg.norm(tl.b - tl.A @ y) <= 1e-11 * np.linalg.norm(tl.b)
