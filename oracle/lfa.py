"""ORACLE (test infrastructure only) — local Fourier analysis of the two-level method
for the multicolour Schwarz order this build runs (readings A4/A5).  SURVEY §8(f) row 2.

LFA looks at the error operator on the infinite grid,

    T = (I - I_q^p A_q^{-1} I_p^q A_p) S_p            (same h, exact second level)

and estimates the asymptotic factor by ρ_2g = sup_θ |T̃(θ)|.  The paper takes the
Schwarz symbols from [nuestropaper2018] (lexicographic block order; not in the container).  The
multicolour order is invariant under translations by D = s + p along every axis, so its LFA is a
*block* LFA: T maps a Bloch wave of quasi-momentum θ (u(x + D e_a) = e^{iθ_a D} u(x)) to another one,
and on the D^d values of one cell it is a D^d × D^d matrix T(θ) — the D^d harmonics θ + 2πk/D
couple.  ρ = sup over θ ∈ (-π/D, π/D]^d of the spectral radius of T(θ), where the cell at θ = 0
drops the constant mode (the kernel of the periodic operator, T 1 = 1), which LFA excludes; its other
D^d - 1 harmonics are genuine frequencies.  Parity pins (tests/test_oracle_lfa.py): stencils against
the assembled matrices and closed forms, the Bloch cells against a brute-force periodic torus, and the
paper's claim that LFA predicts the measured factor against the Dirichlet oracle.

Everything is on the uniform infinite grid with h = 1 (the factor is h-invariant: A_p, A_q scale
alike and the lumped L2 restriction is scale-free).  Basis functions are the cardinal B-splines
B_p(x - j) (P:99-113 on uniform knots), so every operator is a convolution:

    A_p = Σ_a ⊗ (K on axis a, M on the others)         (the tensor form)
    I_p^q = diag(lumped M_q)^{-1} M_qp,  I_q^p = (I_p^q)^T   (lumped L2 projection)
    S_p: colour by colour (c_a mod D), every block x <- x + V_B^T A_B^{-1} V_B (b - A x)

Three analyses:
  * ρ_2g    — two-grid, exact q-level solve at the same h (Table 1's setting);
  * ρ_3g    — three-grid: the q-level system is solved by one two-grid cycle
              M = S_q (I - I_2h^h A_{q,2h}^{-1} I_h^2h A_q) S_q (ν1 = ν2 = 1) with an exact third level;
  * ρ_2g^ag — aggressive two-grid: the second level is degree q on H = 2h, transfers
              R_ag = (I_h^2h) I_p^q, P_ag = R_ag^T (readings A8/A9).
The h <-> 2h transfers couple the 2h-harmonics θ, θ - π; on a Bloch cell of L points
(L a multiple of D, 2 and q+1) the coarse level is a cell of L/2 points and the coupling is exact.
I_2h^h is the knot-insertion embedding B_q(x/2 - J) = Σ_k 2^{-q} C(q+1, k) B_q(x - 2J - k) (reading A8),
I_h^2h its plain transpose; A_{q,2h} is rediscretised on 2h (reading A10; pinned equal to the Galerkin
product).  The q-level smoother is the (q+1)^d-colour Gauss-Seidel (reading A11).
"""
from math import comb

import numpy as np

from .bspline import basis, basis_deriv, gauss_rule


def _cardinal(deg, x, der=False):
    """B_deg(x) (or its derivative) of the cardinal B-spline on knots 0, 1, ..., deg+1."""
    kn = np.arange(deg + 2, dtype=float)
    return (basis_deriv(kn, deg, x) if der else basis(kn, deg, x))[:, 0]


def _integrate(f, lo, hi, nq=12):
    """∫_lo^hi f over unit spans with an nq-point Gauss rule per span (exact for the polynomials here)."""
    gx, gw = gauss_rule(nq, 0.0, 1.0)
    gx, gw = np.asarray(gx), np.asarray(gw)
    return sum(float(np.dot(gw, f(a + gx))) for a in range(lo, hi))


def stencils_1d(p, q):
    """Convolution stencils (dicts offset -> value) at h = 1:
    kp(δ) = ∫ B_p' B_p'(·-δ), mp(δ) = ∫ B_p B_p(·-δ), kq, mq likewise for degree q,
    cqp(δ) = ∫ B_q B_p(·-δ)  (row i of M_qp has cqp(j - i) in column j)."""
    def pair(d1, d2, der, delta):
        lo, hi = min(0, delta) - 1, max(d1, d2 + delta) + 2
        return _integrate(lambda x: _cardinal(d1, x, der) * _cardinal(d2, x - delta, der), lo, hi)
    kp = {d: pair(p, p, True, d) for d in range(-p, p + 1)}
    mp = {d: pair(p, p, False, d) for d in range(-p, p + 1)}
    kq = {d: pair(q, q, True, d) for d in range(-q, q + 1)}
    mq = {d: pair(q, q, False, d) for d in range(-q, q + 1)}
    cqp = {d: pair(q, p, False, d) for d in range(-p - 1, q + 2)}
    return kp, mp, kq, mq, cqp


def bloch_1d(L, st, theta):
    """L x L Bloch matrix of a convolution stencil: (A u)(i) = Σ_δ st(δ) u(i+δ) for u(x+L) = e^{iθL} u(x)."""
    A = np.zeros((L, L), dtype=complex)
    for i in range(L):
        for d, v in st.items():
            j = i + d
            A[i, j % L] += v * np.exp(1j * theta * L * (j // L))
    return A


def _kron_axes(mats):
    """⊗ over axes, axis 0 (x) fastest in the flattened index: kron(m_{d-1}, ..., m_0)."""
    out = mats[-1]
    for m in reversed(mats[:-1]):
        out = np.kron(out, m)
    return out


def _stiffness(L, k, m, theta):
    d = len(theta)
    K = [bloch_1d(L, k, t) for t in theta]
    M = [bloch_1d(L, m, t) for t in theta]
    return sum(_kron_axes([K[a] if b == a else M[b] for b in range(d)]) for a in range(d))


def _block_matrix(s, d, k, m):
    """A_B of an s^d block on the infinite grid (real): Σ_a ⊗(K_B on axis a, M_B elsewhere)."""
    KB = np.array([[k.get(j - i, 0.0) for j in range(s)] for i in range(s)])
    MB = np.array([[m.get(j - i, 0.0) for j in range(s)] for i in range(s)])
    return sum(_kron_axes([KB if b == a else MB for b in range(d)]) for a in range(d))


def error_operator(p, q, s, d, theta, cells=1, st=None):
    """T(θ) on a Bloch cell of L = cells * D points per axis (D = s + p): the two-grid error operator
     with the multicolour smoother (A4/A5) and the exact q-level solve at the same h."""
    kp, mp, kq, mq, cqp = st if st is not None else stencils_1d(p, q)
    D, w = s + p, (s - 1) // 2
    L = cells * D
    N = L ** d
    A = _stiffness(L, kp, mp, theta)
    Aq = _stiffness(L, kq, mq, theta)
    lump = sum(mq.values())                                  # row sum of M_q (lumping)
    R1 = [bloch_1d(L, cqp, t) / lump for t in theta]
    R = _kron_axes(R1)
    P = R.conj().T                                           # I_q^p = (I_p^q)^T on Bloch waves
    AB = _block_matrix(s, d, kp, mp)
    E = np.eye(N, dtype=complex)
    offs = np.array(np.meshgrid(*[np.arange(-w, w + 1)] * d, indexing="ij")).reshape(d, -1)[::-1]  # x fastest
    for col in range(D ** d):                                # colours ascending, c = Σ (c_a mod D) D^a
        cc = [(col // D ** a) % D for a in range(d)]
        for cell in range(cells ** d):
            centre = [cc[a] + D * ((cell // cells ** a) % cells) for a in range(d)]
            pts = np.array(centre)[:, None] + offs           # block points on the infinite grid
            wrap = np.floor_divide(pts, L)
            idx = sum(np.mod(pts[a], L) * L ** a for a in range(d))
            ph = np.exp(1j * sum(theta[a] * L * wrap[a] for a in range(d)))   # u(x) = ph * u(x mod L)
            r = -(A[idx, :] @ E) * ph[:, None]               # V_B (0 - A e) at the true points
            E[idx, :] += np.linalg.solve(AB, r) * ph.conj()[:, None]
    if np.allclose(theta, 0.0):                              # periodic: A_q 1 = 0, use the pseudo-inverse
        C = np.eye(N) - P @ np.linalg.pinv(Aq) @ R @ A
    else:
        C = np.eye(N) - P @ np.linalg.solve(Aq, R @ A)
    return C @ E


def spectrum(p, q, s, d, theta, cells=1, st=None):
    """Eigenvalues of T(θ); at θ = 0 the constant mode (T 1 = 1: A_p 1 = 0) is removed, as in LFA."""
    lam = np.linalg.eigvals(error_operator(p, q, s, d, theta, cells=cells, st=st))
    if np.allclose(theta, 0.0):
        lam = np.delete(lam, np.argmin(np.abs(lam - 1.0)))
    return lam


def rho_2g(p, q, s, d, nk=8, cells=1):
    """ρ_2g ≈ max over the nk^d grid θ_a ∈ {-π/L + 2πj/(nk L)}, j = 1..nk (edges and, for even nk,
    θ = 0 with its constant mode removed), of ρ(T(θ))."""
    L = cells * (s + p)
    st = stencils_1d(p, q)
    ks = np.linspace(-1.0, 1.0, nk + 1)[1:]
    best = 0.0
    for t in np.array(np.meshgrid(*[ks] * d, indexing="ij")).reshape(d, -1).T:
        lam = spectrum(p, q, s, d, list(np.pi / L * t), cells=cells, st=st)
        best = max(best, float(np.max(np.abs(lam))))
    return best


# ---------------------------------------------------------------------------------------------
# three-grid and aggressive two-grid analyses: 2h-harmonics coupled on a Bloch cell
# ---------------------------------------------------------------------------------------------
def mesh_prolong_bloch(L, q, theta):
    """L x L/2 Bloch matrix of I_2h^h (fine u(i) = Σ_J 2^{-q} C(q+1, i - 2J) U(J)) for fine waves
    u(x + L) = e^{iθL} u(x) and coarse waves U(J + L/2) = e^{iθL} U(J) (the same physical wave)."""
    Lc = L // 2
    P = np.zeros((L, Lc), dtype=complex)
    for i in range(L):
        for k in range(q + 2):
            if (i - k) % 2:
                continue
            J = (i - k) // 2
            P[i, J % Lc] += comb(q + 1, k) / 2.0 ** q * np.exp(1j * theta * L * (J // Lc))
    return P


def _cell(p, q, s):
    """Smallest Bloch cell side that is a multiple of D = s + p (the smoother's period), of 2 (the
    coarse mesh) and of q + 1 (the q-level colour period)."""
    D = s + p
    L = D
    while L % 2 or L % (q + 1):
        L += D
    return L


def _schwarz_error(p, s, d, L, theta, kp, mp, A):
    """Error operator of one multicolour Schwarz sweep S_p (A4/A5) on the Bloch cell."""
    D, w = s + p, (s - 1) // 2
    N = L ** d
    cells = L // D
    AB = _block_matrix(s, d, kp, mp)
    E = np.eye(N, dtype=complex)
    offs = np.array(np.meshgrid(*[np.arange(-w, w + 1)] * d, indexing="ij")).reshape(d, -1)[::-1]
    for col in range(D ** d):
        cc = [(col // D ** a) % D for a in range(d)]
        for cell in range(cells ** d):
            centre = [cc[a] + D * ((cell // cells ** a) % cells) for a in range(d)]
            pts = np.array(centre)[:, None] + offs
            wrap = np.floor_divide(pts, L)
            idx = sum(np.mod(pts[a], L) * L ** a for a in range(d))
            ph = np.exp(1j * sum(theta[a] * L * wrap[a] for a in range(d)))
            r = -(A[idx, :] @ E) * ph[:, None]
            E[idx, :] += np.linalg.solve(AB, r) * ph.conj()[:, None]
    return E


def _gs_sweep(X, Rhs, Aq, q, d, L):
    """One (q+1)^d-colour Gauss-Seidel sweep (A11) on the Bloch cell: x_i += (b_i - (A x)_i) / a_ii,
    colour(c) = Σ_a (c_a mod (q+1)) (q+1)^a ascending; X, Rhs are N x k (k right-hand sides)."""
    N = L ** d
    idx = np.arange(N)
    col = sum(((idx // L ** a) % L % (q + 1)) * (q + 1) ** a for a in range(d))
    dg = np.real(np.diag(Aq))
    for c in range((q + 1) ** d):
        pts = idx[col == c]
        X[pts, :] += (Rhs[pts, :] - Aq[pts, :] @ X) / dg[pts, None]
    return X


def _coarse_2h(q, d, theta, L, kq, mq):
    """A_{q,2h} rediscretised on the coarse cell (L/2 points, coarse quasi-momentum 2θ): 1D stencils
    K(2h) = K(h)/2, M(2h) = 2 M(h) (reading A10)."""
    Lc = L // 2
    k2 = {dd: v / 2.0 for dd, v in kq.items()}
    m2 = {dd: 2.0 * v for dd, v in mq.items()}
    return _stiffness(Lc, k2, m2, [2.0 * t for t in theta])


def _solve_or_pinv(A, B, theta):
    if np.allclose(theta, 0.0):                                # periodic constant mode (LFA excludes it)
        return np.linalg.pinv(A) @ B
    return np.linalg.solve(A, B)


def error_operator_ag(p, q, s, d, theta, st=None):
    """T_{p,h}^{q,2h} = (I - P_ag A_{q,2h}^{-1} R_ag A_p) S_p, R_ag = I_h^2h I_p^q."""
    kp, mp, kq, mq, cqp = st if st is not None else stencils_1d(p, q)
    L = _cell(p, q, s)
    N = L ** d
    A = _stiffness(L, kp, mp, theta)
    lump = sum(mq.values())
    R1 = [(mesh_prolong_bloch(L, q, t).conj().T) @ (bloch_1d(L, cqp, t) / lump) for t in theta]
    R = _kron_axes(R1)
    P = R.conj().T
    A2 = _coarse_2h(q, d, theta, L, kq, mq)
    C = np.eye(N) - P @ _solve_or_pinv(A2, R @ A, theta)
    return C @ _schwarz_error(p, s, d, L, theta, kp, mp, A)


def error_operator_3g(p, q, s, d, theta, st=None):
    """M_{p,h}^{q,2h} = (I - I_q^p B_q I_p^q A_p) S_p with B_q = (I - M_q) A_q^{-1} the
    q-level two-grid cycle with zero initial guess: pre-GS, residual, I_h^2h, exact A_{q,2h}, I_2h^h,
    post-GS (ν1 = ν2 = 1)."""
    kp, mp, kq, mq, cqp = st if st is not None else stencils_1d(p, q)
    L = _cell(p, q, s)
    N = L ** d
    A = _stiffness(L, kp, mp, theta)
    Aq = _stiffness(L, kq, mq, theta)
    lump = sum(mq.values())
    R = _kron_axes([bloch_1d(L, cqp, t) / lump for t in theta])
    Pd = R.conj().T
    Pm = _kron_axes([mesh_prolong_bloch(L, q, t) for t in theta])
    A2 = _coarse_2h(q, d, theta, L, kq, mq)
    I = np.eye(N, dtype=complex)
    X = _gs_sweep(np.zeros((N, N), dtype=complex), I, Aq, q, d, L)          # B_q, column by column
    X += Pm @ _solve_or_pinv(A2, Pm.conj().T @ (I - Aq @ X), theta)
    Bq = _gs_sweep(X, I, Aq, q, d, L)
    C = np.eye(N) - Pd @ Bq @ R @ A
    return C @ _schwarz_error(p, s, d, L, theta, kp, mp, A)


def _rho(op, p, q, s, d, nk):
    """max over θ_a ∈ {-π/L + 2πj/(nk L)}, j = 1..nk, of ρ(op(θ)); at θ = 0 the constant mode
    (eigenvalue 1) is removed."""
    L = _cell(p, q, s)
    st = stencils_1d(p, q)
    ks = np.linspace(-1.0, 1.0, nk + 1)[1:]
    best = 0.0
    for t in np.array(np.meshgrid(*[ks] * d, indexing="ij")).reshape(d, -1).T:
        th = list(np.pi / L * t)
        lam = np.linalg.eigvals(op(p, q, s, d, th, st=st))
        if np.allclose(th, 0.0):
            lam = np.delete(lam, np.argmin(np.abs(lam - 1.0)))
        best = max(best, float(np.max(np.abs(lam))))
    return best


def rho_3g(p, q, s, d, nk=4):
    """ρ_3g = sup_θ ρ(M̃(θ))."""
    return _rho(error_operator_3g, p, q, s, d, nk)


def rho_2g_ag(p, q, s, d, nk=4):
    """ρ_2g^ag = sup_θ ρ(T̃_{p,h}^{q,2h}(θ))."""
    return _rho(error_operator_ag, p, q, s, d, nk)
