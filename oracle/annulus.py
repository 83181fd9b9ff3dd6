"""ORACLE (test infrastructure only) — the quarter-annulus NURBS problem.

Domain Ω = {r² <= x² + y² <= R², x, y >= 0}, r = 0.3, R = 0.5; -Δu = f, u = 0 on ∂Ω, with f
such that u = sin(πx) sin(πy)(x² + y² - r²)(x² + y² - R²).

Geometry: the exact quarter circle is the rational quadratic arc with control points
(1,0), (1,1), (0,1) and weights 1, √2/2, 1 on the knots [0,0,0,1,1,1] (angular parameter ξ); the radial
parameter η is linear, ρ(η) = r + (R - r) η.  F(ξ, η) = ρ(η) c(ξ).
Discrete space: NURBS of degree p with maximal smoothness on m uniform spans per direction.
k-refining the geometry keeps its weight function W(ξ) = Σ ω N^2(ξ); the degree-p NURBS basis is
R_i(ξ) = w_i N_i^p(ξ) / W(ξ) with w the coefficients of W in the degree-p basis (radial direction: plain
B-splines, unit weights), φ_ij = R_i(ξ) N_j(η).  Dirichlet: the first and last function in each
direction are removed (as on the square).

Everything below is assembled ELEMENT BY ELEMENT in 2D from the geometry map F, its Jacobian and the
NURBS basis (physical gradients J^{-T} ∇_(ξ,η), weights det J) with a (p+3)^2 Gauss rule per element
(the integrands are rational: the rule is not exact, reading A29 in DESIGN.md).  The second level is the
same construction with degree q = 2 (the geometry's degree) on H = 2h (the improved method, P:263,
reading A1); transfers are the lumped L2 projection and the exact nested embedding between
the q-levels (reading A8), all assembled in 2D.
"""
import functools

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .bspline import basis, basis_deriv, gauss_rule, knot_vector, span_basis
from .multigrid import _colour_sets
from .schwarz import Schwarz

R_IN, R_OUT = 0.3, 0.5
ARC_PTS = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
ARC_W = np.array([1.0, np.sqrt(2.0) / 2.0, 1.0])
ARC_KNOTS = np.array([0.0, 0.0, 0.0, 1.0, 1.0, 1.0])


def arc(xi):
    """Unit quarter-circle arc c(ξ) and c'(ξ) (rational quadratic NURBS)."""
    xi = np.atleast_1d(np.asarray(xi, dtype=float))
    N, dN = basis(ARC_KNOTS, 2, xi), basis_deriv(ARC_KNOTS, 2, xi)
    W, dW = N @ ARC_W, dN @ ARC_W
    num, dnum = N @ (ARC_W[:, None] * ARC_PTS), dN @ (ARC_W[:, None] * ARC_PTS)
    c = num / W[:, None]
    dc = (dnum * W[:, None] - num * dW[:, None]) / W[:, None] ** 2
    return c, dc


def arc_weight(xi):
    """The geometry's weight function W(ξ) = Σ ω_i N_i^2(ξ) and W'(ξ)."""
    xi = np.atleast_1d(np.asarray(xi, dtype=float))
    return basis(ARC_KNOTS, 2, xi) @ ARC_W, basis_deriv(ARC_KNOTS, 2, xi) @ ARC_W


def geometry(xi, eta):
    """F(ξ, η) = ρ(η) c(ξ) and its Jacobian [[x_ξ, x_η], [y_ξ, y_η]] at the points (ξ_k, η_k)."""
    c, dc = arc(xi)
    rho = R_IN + (R_OUT - R_IN) * np.asarray(eta, dtype=float)
    X = rho[:, None] * c
    J = np.empty((len(rho), 2, 2))
    J[:, :, 0] = rho[:, None] * dc
    J[:, :, 1] = (R_OUT - R_IN) * c
    return X, J


@functools.lru_cache(maxsize=None)
def nurbs_weights(p, m):
    """Coefficients w of W(ξ) in the degree-p, C^{p-1} B-spline basis on m uniform spans (W is a
    polynomial of degree 2 <= p, so it lies in the space): L2 projection, exact up to rounding."""
    xi = knot_vector(p, m)
    nf = m + p
    Mm = np.zeros((nf, nf))
    rhs = np.zeros(nf)
    for e in range(m):
        xs, ws = gauss_rule(p + 3, e / m, (e + 1) / m)
        xs, ws = np.asarray(xs), np.asarray(ws)
        Nl = span_basis(xi, p, e, xs)
        Mm[e:e + p + 1, e:e + p + 1] += Nl.T @ (ws[:, None] * Nl)
        rhs[e:e + p + 1] += Nl.T @ (ws * arc_weight(xs)[0])
    return np.linalg.solve(Mm, rhs)


def nurbs_1d(p, m, xs, e):
    """R_i(ξ) = w_i N_i / W and dR_i/dξ at points xs of span e: the p+1 functions alive there
    (full 0-based indices e..e+p), W = Σ w_j N_j from the refined weights."""
    xi = knot_vector(p, m)
    w = nurbs_weights(p, m)[e:e + p + 1]
    N, dN = span_basis(xi, p, e, xs), span_basis(xi, p, e, xs, deriv=True)
    W, dW = N @ w, dN @ w
    R = N * w[None, :] / W[:, None]
    dR = (dN * w[None, :] * W[:, None] - N * w[None, :] * dW[:, None]) / W[:, None] ** 2
    return R, dR


def exact_u(x, y):
    t = x * x + y * y
    return np.sin(np.pi * x) * np.sin(np.pi * y) * (t - R_IN ** 2) * (t - R_OUT ** 2)


def source_f(x, y):
    """f = -Δu for u = s g, s = sin(πx) sin(πy), g = (t - r²)(t - R²), t = x² + y²:
    Δu = g Δs + 2 ∇s·∇g + s Δg, Δs = -2π² s, ∇g = g'(t) (2x, 2y), Δg = 8t + 4 g'(t), g' = 2t - r² - R²."""
    t = x * x + y * y
    s = np.sin(np.pi * x) * np.sin(np.pi * y)
    g = (t - R_IN ** 2) * (t - R_OUT ** 2)
    g1 = 2 * t - R_IN ** 2 - R_OUT ** 2
    sx = np.pi * np.cos(np.pi * x) * np.sin(np.pi * y)
    sy = np.pi * np.sin(np.pi * x) * np.cos(np.pi * y)
    lap = -2 * np.pi ** 2 * s * g + 2 * g1 * 2 * (x * sx + y * sy) + s * (8 * t + 4 * g1)
    return -lap


def assemble(p, m, q=None, want=("A",)):
    """Element-by-element 2D assembly on m x m elements of the degree-p NURBS space (constrained).
    want ⊂ {"A" stiffness, "M" mass, "b" load, "C" cross mass with the degree-q space on the same
    mesh (rows q, cols p), "Mq_full" unconstrained degree-q mass}.  Returns a dict."""
    n1 = m + p - 2
    xi_k = knot_vector(p, m)
    nq = p + 3
    out = {}
    rows, cols, vA, vM, vC = [], [], [], [], []
    b = np.zeros(n1 * n1)
    crow, ccol = [], []
    if q is not None:
        n1q = m + q - 2
    for ey in range(m):
        ys, wy = gauss_rule(nq, ey / m, (ey + 1) / m)
        ys, wy = np.asarray(ys), np.asarray(wy)
        Ny, dNy = span_basis(xi_k, p, ey, ys), span_basis(xi_k, p, ey, ys, deriv=True)
        if q is not None:
            Nyq = span_basis(knot_vector(q, m), q, ey, ys)
        for ex in range(m):
            xs, wx = gauss_rule(nq, ex / m, (ex + 1) / m)
            xs, wx = np.asarray(xs), np.asarray(wx)
            Rx, dRx = nurbs_1d(p, m, xs, ex)
            XI, ETA = np.meshgrid(xs, ys, indexing="xy")          # [iy, ix] points
            X, J = geometry(XI.ravel(), ETA.ravel())
            det = np.abs(J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0])   # |det J| (F reverses orientation)
            Jinv = np.linalg.inv(J)                                 # [k, 2, 2]
            wq = (wy[:, None] * wx[None, :]).ravel() * det
            # local functions (ix local in x, iy local in y), x fastest
            phi = np.einsum("yj,xi->yxji", Ny, Rx).reshape(len(ys) * len(xs), -1)
            dxi = np.einsum("yj,xi->yxji", Ny, dRx).reshape(len(ys) * len(xs), -1)
            deta = np.einsum("yj,xi->yxji", dNy, Rx).reshape(len(ys) * len(xs), -1)
            # physical gradient = J^{-T} (d/dξ, d/dη)
            gx = Jinv[:, 0, 0][:, None] * dxi + Jinv[:, 1, 0][:, None] * deta
            gy = Jinv[:, 0, 1][:, None] * dxi + Jinv[:, 1, 1][:, None] * deta
            gi = np.array([(ey + jy - 1) * n1 + (ex + ix - 1) for jy in range(p + 1) for ix in range(p + 1)])
            ok = np.array([0 <= ex + ix - 1 < n1 and 0 <= ey + jy - 1 < n1 for jy in range(p + 1) for ix in range(p + 1)])
            sel = np.nonzero(ok)[0]
            G = gi[sel]
            if "A" in want:
                Ae = gx[:, sel].T @ (wq[:, None] * gx[:, sel]) + gy[:, sel].T @ (wq[:, None] * gy[:, sel])
                rows.append(np.repeat(G, len(G))); cols.append(np.tile(G, len(G))); vA.append(Ae.ravel())
            if "M" in want:
                Me = phi[:, sel].T @ (wq[:, None] * phi[:, sel])
                vM.append(Me.ravel())
                if "A" not in want:
                    rows.append(np.repeat(G, len(G))); cols.append(np.tile(G, len(G)))
            if "b" in want:
                b[G] += phi[:, sel].T @ (wq * source_f(X[:, 0], X[:, 1]))
            if "C" in want:
                Rxq, _ = nurbs_1d(q, m, xs, ex)
                phq = np.einsum("yj,xi->yxji", Nyq, Rxq).reshape(len(ys) * len(xs), -1)
                giq = np.array([(ey + jy - 1) * n1q + (ex + ix - 1) for jy in range(q + 1) for ix in range(q + 1)])
                okq = np.array([0 <= ex + ix - 1 < n1q and 0 <= ey + jy - 1 < n1q
                                for jy in range(q + 1) for ix in range(q + 1)])
                sq = np.nonzero(okq)[0]
                Ce = phq[:, sq].T @ (wq[:, None] * phi[:, sel])
                crow.append(np.repeat(giq[sq], len(G))); ccol.append(np.tile(G, len(sq))); vC.append(Ce.ravel())
    N = n1 * n1
    if "A" in want:
        out["A"] = sp.csr_matrix((np.concatenate(vA), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))
    if "M" in want:
        out["M"] = sp.csr_matrix((np.concatenate(vM), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))
    if "b" in want:
        out["b"] = b
    if "C" in want:
        out["C"] = sp.csr_matrix((np.concatenate(vC), (np.concatenate(crow), np.concatenate(ccol))),
                                 shape=(n1q * n1q, N))
    return out


def lumped_q_mass(q, m):
    """D_ii = ∫_Ω φ^q_i dx (= row sums of the UNCONSTRAINED degree-q mass: the unconstrained NURBS basis
    is a partition of unity, reading A6), at the constrained rows."""
    n1 = m + q - 2
    D = np.zeros(n1 * n1)
    for ey in range(m):
        ys, wy = gauss_rule(q + 3, ey / m, (ey + 1) / m)
        ys, wy = np.asarray(ys), np.asarray(wy)
        Ny = span_basis(knot_vector(q, m), q, ey, ys)
        for ex in range(m):
            xs, wx = gauss_rule(q + 3, ex / m, (ex + 1) / m)
            xs, wx = np.asarray(xs), np.asarray(wx)
            Rx, _ = nurbs_1d(q, m, xs, ex)
            XI, ETA = np.meshgrid(xs, ys, indexing="xy")
            _, J = geometry(XI.ravel(), ETA.ravel())
            det = np.abs(J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0])   # |det J| (F reverses orientation)
            wq = (wy[:, None] * wx[None, :]).ravel() * det
            phi = np.einsum("yj,xi->yxji", Ny, Rx).reshape(len(ys) * len(xs), -1)
            for jy in range(q + 1):
                for ix in range(q + 1):
                    cx, cy = ex + ix - 1, ey + jy - 1
                    if 0 <= cx < n1 and 0 <= cy < n1:
                        D[cy * n1 + cx] += wq @ phi[:, jy * (q + 1) + ix]
    return D


def embedding(q, mc):
    """The exact nested embedding of the degree-q NURBS space on mc spans into the one on 2 mc spans
    (same weight function W): P = M_h^{-1} M_{h,2h} (2D L2 projection, exact for nested spaces), constrained."""
    mf = 2 * mc
    Mh = assemble(q, mf, want=("M",))["M"].toarray()
    n1f, n1c = mf + q - 2, mc + q - 2
    Mhc = np.zeros((n1f * n1f, n1c * n1c))
    kf, kc = knot_vector(q, mf), knot_vector(q, mc)
    for ey in range(mf):
        ys, wy = gauss_rule(q + 3, ey / mf, (ey + 1) / mf)
        ys, wy = np.asarray(ys), np.asarray(wy)
        Nyf = span_basis(kf, q, ey, ys)
        Nyc = span_basis(kc, q, ey // 2, ys)
        for ex in range(mf):
            xs, wx = gauss_rule(q + 3, ex / mf, (ex + 1) / mf)
            xs, wx = np.asarray(xs), np.asarray(wx)
            Rxf, _ = nurbs_1d(q, mf, xs, ex)
            Rxc, _ = nurbs_1d(q, mc, xs, ex // 2)
            XI, ETA = np.meshgrid(xs, ys, indexing="xy")
            _, J = geometry(XI.ravel(), ETA.ravel())
            det = np.abs(J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0])   # |det J| (F reverses orientation)
            wq = (wy[:, None] * wx[None, :]).ravel() * det
            phf = np.einsum("yj,xi->yxji", Nyf, Rxf).reshape(len(ys) * len(xs), -1)
            phc = np.einsum("yj,xi->yxji", Nyc, Rxc).reshape(len(ys) * len(xs), -1)
            for jy in range(q + 1):
                for ix in range(q + 1):
                    fx, fy = ex + ix - 1, ey + jy - 1
                    if not (0 <= fx < n1f and 0 <= fy < n1f):
                        continue
                    for ky in range(q + 1):
                        for kx in range(q + 1):
                            cx, cy = ex // 2 + kx - 1, ey // 2 + ky - 1
                            if 0 <= cx < n1c and 0 <= cy < n1c:
                                Mhc[fy * n1f + fx, cy * n1c + cx] += wq @ (phf[:, jy * (q + 1) + ix] *
                                                                          phc[:, ky * (q + 1) + kx])
    P = np.linalg.solve(Mh, Mhc)
    P[np.abs(P) < 1e-13] = 0.0
    return sp.csr_matrix(P)


class AnnulusHierarchy:
    """The q-level V(1,1) on the degree-q NURBS space: (q+1)^2-colour Gauss-Seidel (A11),
    embedding P and its unscaled transpose (A8), rediscretised operators (A10), dense solve at m <= 8."""

    def __init__(self, q, m0, coarsest_m=8):
        self.q = q
        self.levels = []
        m = m0
        while True:
            A = assemble(q, m)["A"].tocsr()
            n = m + q - 2
            lev = {"m": m, "n": n, "A": A, "diag": A.diagonal().copy(), "colours": _colour_sets(n, 2, q + 1)}
            self.levels.append(lev)
            if m <= coarsest_m:
                lev["chol"] = sla.cho_factor(A.toarray(), lower=True)
                break
            lev["P"] = embedding(q, m // 2)
            m //= 2

    def gs(self, l, x, b):
        lev = self.levels[l]
        for pts in lev["colours"]:
            x[pts] += (b[pts] - lev["A"][pts] @ x) / lev["diag"][pts]
        return x

    def vcycle(self, b, l=0):
        lev = self.levels[l]
        if "chol" in lev:
            return sla.cho_solve(lev["chol"], b)
        x = np.zeros_like(b)
        self.gs(l, x, b)
        r = b - lev["A"] @ x
        ec = self.vcycle(lev["P"].T @ r, l + 1)
        x += lev["P"] @ ec
        self.gs(l, x, b)
        return x


class AnnulusTwoLevel:
    """Algorithm 1 on the quarter annulus: multicolour Schwarz on the degree-p NURBS level
    (blocks s x s, reading A4), lumped L2 restriction to degree q = 2 on H = 2h composed with the
    embedding (A9), second level exact ("DS", sparse direct) or one V(1,1) ("MG")."""

    def __init__(self, p, m, s, coarse="vcycle", q=2, coarsest_m=8):
        self.p, self.m, self.s, self.q = p, m, s, q
        self.n1 = m + p - 2
        self.N = self.n1 ** 2
        got = assemble(p, m, want=("A", "b"))
        self.A, self.b = got["A"].tocsr(), got["b"]
        self.smoother = Schwarz(self.A, self.n1, 2, s, p, "multicolour")
        C = assemble(p, m, q=q, want=("C",))["C"]                 # degree-q x degree-p cross mass, mesh h
        Rdeg = sp.diags(1.0 / lumped_q_mass(q, m)) @ C            # lumped L2 projection
        self.R = (embedding(q, m // 2).T @ Rdeg).tocsr()          # aggressive: mesh 2h (A9)
        self.RT = self.R.T.tocsr()
        self.Nc = self.R.shape[0]
        if coarse == "vcycle":
            self.mg = AnnulusHierarchy(q, m // 2, coarsest_m)
            self._csolve = self.mg.vcycle
        else:
            import scipy.sparse.linalg as spla
            self._csolve = spla.factorized(assemble(q, m // 2)["A"].tocsc())

    def iterate(self, x, b):
        self.smoother.sweep(x, b)
        x += self.RT @ self._csolve(self.R @ (b - self.A @ x))
        return x

    def solve(self, b, x0, rtol=1e-8, maxit=200):
        x = x0.copy()
        r0 = np.linalg.norm(b - self.A @ x)
        it, r = 0, r0
        while it < maxit and r > rtol * r0:
            self.iterate(x, b)
            it += 1
            r = np.linalg.norm(b - self.A @ x)
        return x, it, r / r0


def l2_error(p, m, coef):
    """||u - u_h||_{L2(Ω)} for u_h = Σ coef_ij φ_ij (constrained coefficients, x fastest)."""
    n1 = m + p - 2
    C = np.zeros((n1 + 2, n1 + 2))
    C[1:-1, 1:-1] = coef.reshape(n1, n1)
    err2 = 0.0
    for ey in range(m):
        ys, wy = gauss_rule(p + 3, ey / m, (ey + 1) / m)
        ys, wy = np.asarray(ys), np.asarray(wy)
        Ny = span_basis(knot_vector(p, m), p, ey, ys)
        for ex in range(m):
            xs, wx = gauss_rule(p + 3, ex / m, (ex + 1) / m)
            xs, wx = np.asarray(xs), np.asarray(wx)
            Rx, _ = nurbs_1d(p, m, xs, ex)
            XI, ETA = np.meshgrid(xs, ys, indexing="xy")
            X, J = geometry(XI.ravel(), ETA.ravel())
            det = np.abs(J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0])   # |det J| (F reverses orientation)
            wq = (wy[:, None] * wx[None, :]).ravel() * det
            uh = np.einsum("yj,xi,ji->yx", Ny, Rx, C[ey:ey + p + 1, ex:ex + p + 1]).ravel()
            err2 += wq @ (exact_u(X[:, 0], X[:, 1]) - uh) ** 2
    return np.sqrt(err2)


def separable_1d(p, m):
    """The four 1D weighted matrices of the tensor structure of A on this geometry (constrained):
    F = ρ(η) c(ξ) with |c| = 1 has orthogonal Jacobian columns ρ c' and ρ' c, |det J| = ρ ρ' s (s = |c'|), so
    a(φ_ik, φ_jl) = ∫ R_i' R_j' / s dξ ∫ N_k N_l ρ'/ρ dη + ∫ R_i R_j s dξ ∫ N_k' N_l' ρ/ρ' dη, i.e.
    A = My ⊗ Kx + Ky ⊗ Mx (x = ξ fastest) with Kx = (R'R'/s), Mx = (R R s), Ky = (N'N' ρ/ρ'), My = (N N ρ'/ρ).
    Same (p+3)-point Gauss rule per span as ``assemble`` (whose 2D rule is its tensor product)."""
    nf = m + p
    Kx, Mx, Ky, My = (np.zeros((nf, nf)) for _ in range(4))
    kv = knot_vector(p, m)
    dr = R_OUT - R_IN
    for e in range(m):
        xs, ws = gauss_rule(p + 3, e / m, (e + 1) / m)
        xs, ws = np.asarray(xs), np.asarray(ws)
        R, dR = nurbs_1d(p, m, xs, e)
        s = np.hypot(*arc(xs)[1].T)
        sl = slice(e, e + p + 1)
        Kx[sl, sl] += dR.T @ ((ws / s)[:, None] * dR)
        Mx[sl, sl] += R.T @ ((ws * s)[:, None] * R)
        N, dN = span_basis(kv, p, e, xs), span_basis(kv, p, e, xs, deriv=True)
        rho = R_IN + dr * xs
        Ky[sl, sl] += dN.T @ ((ws * rho / dr)[:, None] * dN)
        My[sl, sl] += N.T @ ((ws * dr / rho)[:, None] * N)
    c = slice(1, -1)
    return Kx[c, c], Mx[c, c], Ky[c, c], My[c, c]
