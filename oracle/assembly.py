"""ORACLE (test infrastructure only) — Galerkin matrices and load vectors.

Layout: a d-dim constrained index (i_0, …, i_{d-1}), 0 ≤ i_a < n1 = m+p-2,
is flattened x-fastest: g = i_0 + n1 (i_1 + n1 i_2).  Constrained index i_a is the
paper's basis function N_{i_a+2}.

All integrals use Gauss–Legendre with p+1 points per knot span: the
integrands of K and M are polynomials of degree ≤ 2p on each span, so the rule is
exact.  The load uses p+3 points (A17).
"""
import functools

import numpy as np
import scipy.sparse as sp

from .bspline import basis, basis_deriv, knot_vector, span_basis, span_rule


def n_dofs_1d(p, m):
    """dim S_h^p = p + m - 2."""
    return p + m - 2


def _span_tables(p, m, nq):
    """For each span e: quadrature points/weights and the p+1 non-zero functions
    (full 0-based indices e..e+p) with their derivatives at those points."""
    xi = knot_vector(p, m)
    out = []
    for e in range(m):
        xs, ws = span_rule(m, e, nq)
        N = span_basis(xi, p, e, xs)
        dN = span_basis(xi, p, e, xs, deriv=True) if p >= 1 else np.zeros_like(N)
        out.append((xs, ws, N, dN))
    return out


def matrices_1d(p, m, constrained=True):
    """1D stiffness K_{ij} = ∫ N_j' N_i' and mass M_{ij} = ∫ N_j N_i (P:74, P:83 in 1D),
    assembled element by element.  ``constrained`` drops N_1 and N_{m+p} (Dirichlet)."""
    nf = m + p
    K = np.zeros((nf, nf))
    M = np.zeros((nf, nf))
    for e, (xs, ws, N, dN) in enumerate(_span_tables(p, m, p + 1)):
        sl = slice(e, e + p + 1)
        K[sl, sl] += dN.T @ (ws[:, None] * dN)
        M[sl, sl] += N.T @ (ws[:, None] * N)
    if constrained:
        K, M = K[1:-1, 1:-1], M[1:-1, 1:-1]
    return K, M


def cross_mass_1d(q, p, m, constrained=True):
    """(M_p^{q})_{ij} = ∫ φ_i^{q} φ_j^{p} on the same mesh h = 1/m, rows q, cols p."""
    xq, xp = knot_vector(q, m), knot_vector(p, m)
    nq_pts = max(p, q) + 1
    Mc = np.zeros((m + q, m + p))
    for e in range(m):
        xs, ws = span_rule(m, e, nq_pts)
        Nq = span_basis(xq, q, e, xs)
        Np = span_basis(xp, p, e, xs)
        Mc[e:e + q + 1, e:e + p + 1] += Nq.T @ (ws[:, None] * Np)
    if constrained:
        Mc = Mc[1:-1, 1:-1]
    return Mc


def _kron_list(mats):
    """Kronecker product with the LAST list entry fastest (x-fastest when mats = [A_z, A_y, A_x])."""
    return functools.reduce(np.kron, mats)


def stiffness_elementwise(p, m, d, constrained=True):
    """Sparse A_p = (a(φ_j, φ_i)) for φ = tensor-product B-splines,
    assembled element by element on the tensor Gauss rule (p+1)^d.

    Each element's local matrix is Σ_k ∫ ∂_k φ_a ∂_k φ_b, scatter-added into a banded
    global array (offsets t_a = col_a - row_a ∈ [-p, p]), then converted to CSR.
    """
    nf = m + p
    n1 = nf - 2 if constrained else nf
    off = 1 if constrained else 0
    tabs = _span_tables(p, m, p + 1)
    nb = 2 * p + 1
    N = n1 ** d
    band = np.zeros((N, nb ** d))
    loc = np.arange(p + 1)
    # local multi-indices, x fastest
    grids = np.meshgrid(*([loc] * d), indexing="ij")          # grids[a] varies along axis a
    loc_idx = [g.transpose(tuple(range(d))[::-1]).ravel() for g in grids]  # x-fastest flatten
    for elem in np.ndindex(*([m] * d)):                      # elem[a] = span index along axis a
        # gradient tensors: for axis k, product over axes of (dN if a==k else N)
        Wq = _kron_list([tabs[elem[a]][1] for a in reversed(range(d))])
        Kloc = 0.0
        for k in range(d):
            G = _kron_list([(tabs[elem[a]][3] if a == k else tabs[elem[a]][2])
                            for a in reversed(range(d))])
            Kloc = Kloc + G.T @ (Wq[:, None] * G)
        # global (constrained) indices of the local functions
        full = [elem[a] + loc_idx[a] for a in range(d)]
        ok = np.ones(len(loc_idx[0]), dtype=bool)
        gi = np.zeros(len(loc_idx[0]), dtype=np.int64)
        for a in range(d):
            c = full[a] - off
            ok &= (c >= 0) & (c < n1)
            gi += c * n1 ** a
        rows = np.nonzero(ok)[0]
        tcode = np.zeros((len(rows), len(rows)), dtype=np.int64)
        for a in range(d):
            fa = full[a][rows]
            tcode += (fa[None, :] - fa[:, None] + p) * nb ** a
        # (row, offset) pairs are distinct within one element, so plain += is a scatter-add
        band[gi[rows][:, None], tcode] += Kloc[np.ix_(rows, rows)]
    return _band_to_csr(band, n1, p, d)


def _band_to_csr(band, n1, p, d):
    nb = 2 * p + 1
    N = n1 ** d
    rows_all, cols_all, vals_all = [], [], []
    idx = np.arange(N)
    coords = [(idx // n1 ** a) % n1 for a in range(d)]
    for tcode in range(nb ** d):
        t = [(tcode // nb ** a) % nb - p for a in range(d)]
        ok = np.ones(N, dtype=bool)
        col = np.zeros(N, dtype=np.int64)
        for a in range(d):
            c = coords[a] + t[a]
            ok &= (c >= 0) & (c < n1)
            col += c * n1 ** a
        v = band[:, tcode]
        keep = ok & (v != 0.0)
        rows_all.append(idx[keep]); cols_all.append(col[keep]); vals_all.append(v[keep])
    A = sp.csr_matrix((np.concatenate(vals_all), (np.concatenate(rows_all), np.concatenate(cols_all))),
                      shape=(N, N))
    A.sort_indices()
    return A


def stiffness_kron(p, m, d, constrained=True):
    """A_p = Σ_a (⊗_b X_b), X_b = K if b == a else M (tensor-product structure of P:119-127).
    Pinned equal to ``stiffness_elementwise`` in tests; used where element loops are too slow."""
    K, M = matrices_1d(p, m, constrained)
    Ks, Ms = sp.csr_matrix(K), sp.csr_matrix(M)
    A = None
    for a in range(d):
        mats = [Ks if b == a else Ms for b in reversed(range(d))]   # slowest axis first
        T = functools.reduce(lambda u, v: sp.kron(u, v, format="csr"), mats)
        A = T if A is None else A + T
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    A.sort_indices()
    return A


def stiffness(p, m, d, constrained=True, method="auto"):
    """Galerkin stiffness.  ``auto`` = element loop for ≤ 70k elements, else Kronecker."""
    if method == "element" or (method == "auto" and m ** d <= 70000):
        return stiffness_elementwise(p, m, d, constrained)
    return stiffness_kron(p, m, d, constrained)


def sine_f(d):
    """f = d π² ∏ sin(π x_a), so that u = ∏ sin(π x_a) solves -Δu = f (P:401 for d = 2)."""
    return lambda *xs: d * np.pi ** 2 * np.prod([np.sin(np.pi * x) for x in xs], axis=0)


def load_1d_sine(p, m):
    """g_i = ∫_0^1 sin(π x) N_i(x) dx with p+3 Gauss points per span (A17); constrained i."""
    xi = knot_vector(p, m)
    g = np.zeros(m + p)
    for e in range(m):
        xs, ws = span_rule(m, e, p + 3)
        g[e:e + p + 1] += span_basis(xi, p, e, xs).T @ (ws * np.sin(np.pi * xs))
    return g[1:-1]


def load_sine(p, m, d):
    """b_i = (f, φ_i) for f = dπ²∏ sin(π x_a).  f and φ_i are both tensor products and
    the rule is a tensor Gauss rule, so b = dπ² ⊗_a g (pinned against ``load_sine_elementwise``)."""
    g = load_1d_sine(p, m)
    return d * np.pi ** 2 * _kron_list([g] * d)


def load_sine_elementwise(p, m, d):
    """Same integral, element by element on the tensor (p+3)^d rule (small m only)."""
    tabs = _span_tables(p, m, p + 3)
    n1 = m + p - 2
    b = np.zeros(n1 ** d)
    f = sine_f(d)
    loc = np.arange(p + 1)
    for elem in np.ndindex(*([m] * d)):
        pts = np.meshgrid(*[tabs[elem[a]][0] for a in range(d)], indexing="ij")
        W = functools.reduce(np.multiply.outer, [tabs[elem[a]][1] for a in range(d)])
        fw = (f(*pts) * W)                       # indexed [q_0, q_1, ...]
        vals = fw
        for a in range(d):                       # contract quad axis a with N[:, loc]
            vals = np.tensordot(vals, tabs[elem[a]][2], axes=([0], [0]))
        # vals indexed [a_0, a_1, ...] after d contractions (each appended at the end)
        for li in np.ndindex(*([p + 1] * d)):
            c = [elem[a] + li[a] - 1 for a in range(d)]
            if all(0 <= ca < n1 for ca in c):
                b[sum(c[a] * n1 ** a for a in range(d))] += vals[li]
    return b


def l2_error_sine(p, m, d, coef):
    """‖u - u_h‖_{L2} for u = ∏ sin(π x_a), u_h = Σ coef_g φ_g, by element quadrature (p+3 pts)."""
    tabs = _span_tables(p, m, p + 3)
    n1 = m + p - 2
    C = coef.reshape([n1] * d)                   # C[i_{d-1}, ..., i_0] (x fastest)
    Cp = np.zeros([n1 + 2] * d)
    Cp[tuple([slice(1, -1)] * d)] = C
    err2 = 0.0
    for elem in np.ndindex(*([m] * d)):
        pts = np.meshgrid(*[tabs[elem[a]][0] for a in range(d)], indexing="ij")
        W = functools.reduce(np.multiply.outer, [tabs[elem[a]][1] for a in range(d)])
        u = np.prod([np.sin(np.pi * x) for x in pts], axis=0)
        # local coefficient block, axis order [a_{d-1} .. a_0] in Cp -> reverse to [a_0 .. a_{d-1}]
        sl = tuple(slice(elem[a], elem[a] + p + 1) for a in reversed(range(d)))
        cl = np.transpose(Cp[sl], tuple(range(d))[::-1])
        uh = cl
        for a in range(d):
            uh = np.tensordot(uh, tabs[elem[a]][2], axes=([0], [1]))
        err2 += np.sum(W * (u - uh) ** 2)
    return np.sqrt(err2)
