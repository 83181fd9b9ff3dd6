"""Pins of the LFA oracle (oracle/lfa.py): closed forms, the assembled matrices,
a brute-force periodic torus, and the paper's claim that LFA predicts the measured factor."""
import numpy as np
import pytest

from oracle.assembly import cross_mass_1d, matrices_1d
from oracle.lfa import error_operator, rho_2g, spectrum, stencils_1d
from oracle.twolevel import TwoLevel
from synthetic_inputs import initial_guess


def test_stencils_closed_forms():
    """p = 1: K = (-1, 2, -1), M = (1/6, 2/3, 1/6) at h = 1; any p: Σ K = 0 (constants), Σ M = Σ C = 1
    (∫ B_p = 1), symmetric K, M."""
    k, m, _, _, c = stencils_1d(1, 1)
    assert np.allclose([k[-1], k[0], k[1]], [-1, 2, -1], atol=1e-14)
    assert np.allclose([m[-1], m[0], m[1]], [1 / 6, 2 / 3, 1 / 6], atol=1e-14)
    for p in range(1, 7):
        for q in (1, 2):
            k, m, kq, mq, c = stencils_1d(p, q)
            assert abs(sum(k.values())) < 1e-13 and abs(sum(kq.values())) < 1e-13
            assert abs(sum(m.values()) - 1) < 1e-13 and abs(sum(c.values()) - 1) < 1e-13
            assert all(abs(k[d] - k[-d]) < 1e-14 and abs(m[d] - m[-d]) < 1e-14 for d in k)


@pytest.mark.parametrize("p", [2, 3, 5, 8])
def test_stencils_match_assembled_interior_rows(p):
    """The infinite-grid stencils are the interior rows of the assembled 1D matrices
    scaled to h = 1 (K h, M / h), and an interior row of the cross mass M_qp is a shifted
    copy of cqp."""
    mm = 40
    K, M = matrices_1d(p, mm)
    k, m, _, _, c = stencils_1d(p, 1)
    i = K.shape[0] // 2
    for d in range(-p, p + 1):
        assert abs(K[i, i + d] / mm - k[d]) < 1e-12
        assert abs(M[i, i + d] * mm - m[d]) < 1e-12
    C = cross_mass_1d(1, p, mm) * mm
    row = C[C.shape[0] // 2]
    nz = np.nonzero(np.abs(row) > 1e-15)[0]
    vals = [c[d] for d in sorted(c) if abs(c[d]) > 1e-15]
    assert np.allclose(row[nz[0]:nz[-1] + 1], vals, atol=1e-12)


def _torus_spectrum(p, q, s, L):
    """Brute force: the real periodic torus of L x L cardinal B-splines, the multicolour sweep block by
    block, exact q-level solve by pseudo-inverse; all eigenvalues of the dense error operator."""
    k, m, kq, mq, c = stencils_1d(p, q)

    def circ(st):
        A = np.zeros((L, L))
        for i in range(L):
            for d, v in st.items():
                A[i, (i + d) % L] += v
        return A
    K1, M1, Kq1, Mq1, C1 = circ(k), circ(m), circ(kq), circ(mq), circ(c)
    A = np.kron(K1, M1) + np.kron(M1, K1)
    Aq = np.kron(Kq1, Mq1) + np.kron(Mq1, Kq1)
    R1 = np.diag(1.0 / Mq1.sum(1)) @ C1
    R = np.kron(R1, R1)
    N, w, D = L * L, (s - 1) // 2, s + p
    E = np.eye(N)
    for c1 in range(D):
        for c0 in range(D):
            for cy in range(c1, L, D):
                for cx in range(c0, L, D):
                    idx = [((cy + a) % L) * L + (cx + b) % L for a in range(-w, w + 1) for b in range(-w, w + 1)]
                    E[idx, :] -= np.linalg.solve(A[np.ix_(idx, idx)], A[idx, :] @ E)
    T = (np.eye(N) - R.T @ np.linalg.pinv(Aq) @ R @ A) @ E
    return np.linalg.eigvals(T)


@pytest.mark.parametrize("p,s", [(2, 3), (3, 3)])
def test_bloch_cells_equal_brute_force_torus(p, s):
    """A torus of L = 2D points per axis has exactly the Bloch momenta θ_a ∈ {0, π/D}: the union of the
    cell spectra T(θ) must be the torus spectrum (each cell eigenvalue found in it), and the cell at
    θ = 0 carries the constant mode (eigenvalue 1)."""
    D = s + p
    mu = _torus_spectrum(p, 1, s, 2 * D)
    th = [0.0, np.pi / D]
    worst = 0.0
    for ty in th:
        for tx in th:
            lam = np.linalg.eigvals(error_operator(p, 1, s, 2, [tx, ty]))
            worst = max(worst, max(float(np.min(np.abs(mu - l))) for l in lam))
    assert worst < 1e-9
    lam0 = np.linalg.eigvals(error_operator(p, 1, s, 2, [0.0, 0.0]))
    assert np.min(np.abs(lam0 - 1.0)) < 1e-10
    assert np.max(np.abs(spectrum(p, 1, s, 2, [0.0, 0.0]))) < 0.999


def test_cells_consistent_across_cell_sizes():
    """A 2-cell Bloch block at θ carries the 1-cell spectra at θ and θ + π/D (per axis)."""
    p, s = 2, 3
    D = s + p
    t = [0.3 / D, -0.7 / D]
    lam2 = np.linalg.eigvals(error_operator(p, 1, s, 2, t, cells=2))
    for sx in (0.0, np.pi / D):
        for sy in (0.0, np.pi / D):
            lam1 = np.linalg.eigvals(error_operator(p, 1, s, 2, [t[0] + sx, t[1] + sy]))
            assert max(float(np.min(np.abs(lam2 - l))) for l in lam1) < 1e-9


@pytest.mark.parametrize("p,s", [(2, 3), (3, 3), (4, 3), (5, 5)])
def test_lfa_predicts_measured_factor(p, s):
    """the LFA factor predicts the measured one (Table 1 shows |ρ_2g - ρ_h| ≤ 0.022).  Here:
    block LFA of the multicolour two-grid (exact q = 1 solve at the same h) against the Dirichlet
    oracle's measured asymptotic factor (b = 0, random start), m = 32."""
    lfa = rho_2g(p, 1, s, 2, nk=4)
    tl = TwoLevel(2, p, 1, 32, s=s, coarse="exact", h_factor=1, order="multicolour")
    rho, _ = tl.rate(initial_guess(tl.N), iters=40, last=10)
    assert abs(lfa - rho) < 0.03, (lfa, rho)
