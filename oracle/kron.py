"""ORACLE (test infrastructure only) — Algorithm 1 at full BASELINE sizes, without assembling A_p.

The sparse d-dim stiffness of C3-C5 does not fit a test box (C4: 736M non-zeros, C5: 23G), and the
sequential block loop of ``schwarz.Schwarz`` is too slow there.  This module computes the SAME
iteration as ``twolevel.TwoLevel(order="multicolour")`` with two substitutions, both pinned against
``TwoLevel`` / ``assembly.stiffness`` in ``tests/test_oracle_kron.py``:

1. The operator is applied from its tensor-product form:
       A_p = Σ_a ⊗_b X_b,   X_b = K (1D stiffness) if b == a else M (1D mass),
   each term as d plain 1D matrix products along the axes (no factor shared between terms), with
   the oracle's own 1D matrices ``assembly.matrices_1d``.  Block matrices A^B = V_B A V_B^T
   are the same sums of Kronecker products of the 1D sub-blocks X[B_a, B_a].
2. The multicolour sweep (reading A4) is run colour by colour: every block of colour c is computed
   from the x left by colour c-1 and the corrections are then added.  Same-colour blocks are
   A-decoupled and disjoint, so this equals the sequential sweep in colour-major order (pinned in
   tests/test_oracle_schwarz.py for ``Schwarz.colour_step_parallel``).  Local solves are dense LU
   (``numpy.linalg.solve``) of the assembled block; while all block inverses fit
   in ``cache_bytes`` they are formed once (``numpy.linalg.inv``) and reused by later sweeps.

Transfers are the 1D factors of ``transfer.restriction`` applied axis by axis (R = ⊗ R1, P:220,
P:300); the second level is ``multigrid.QHierarchy`` (one V(1,1)) or an exact sparse
solve of the rediscretised A_q.
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .assembly import matrices_1d, stiffness
from .multigrid import QHierarchy
from .transfer import degree_restriction_1d, mesh_prolongation_1d


def axis_apply(X, arr, a, d):
    """out[..., i_a, ...] = Σ_j X[i_a, j] arr[..., j, ...] along grid axis a (axis 0 = x, fastest).
    ``arr`` has array shape [n_{d-1}, ..., n_0] (C order, x fastest)."""
    ax = d - 1 - a
    t = np.moveaxis(arr, ax, 0)
    sh = t.shape
    out = X @ t.reshape(sh[0], -1)
    return np.moveaxis(np.asarray(out).reshape((X.shape[0],) + sh[1:]), 0, ax)


def kron_apply(mats, x, n_in, d):
    """(⊗_a mats[a]) x, mats[a] acting on grid axis a; x flat (x fastest) with n_in per axis."""
    arr = x.reshape([n_in] * d)
    for a in range(d):
        arr = axis_apply(mats[a], arr, a, d)
    return np.ascontiguousarray(arr).ravel()


class KronOperator:
    """y = A_p x, A_p = Σ_a ⊗_b (K if b == a else M)."""

    def __init__(self, p, m, d):
        self.p, self.m, self.d = p, m, d
        self.n1 = m + p - 2
        K, M = matrices_1d(p, m)
        self.Kd, self.Md = K, M
        self.K, self.M = sp.csr_matrix(K), sp.csr_matrix(M)

    def apply(self, x):
        y = np.zeros(self.n1 ** self.d)
        for a in range(self.d):
            y += kron_apply([self.K if b == a else self.M for b in range(self.d)], x, self.n1, self.d)
        return y


def _colour_groups(n1, d, s, D, colour):
    """Blocks of one colour grouped by clipped shape: list of (lo (nb, d), ln (d,)).
    Centres c_a ≡ colour digit a (mod D) (reading A5); window [c_a - w, c_a + w] ∩ [0, n1) (A3)."""
    w = (s - 1) // 2
    digits = [(colour // D ** a) % D for a in range(d)]
    axes = [np.arange(dg, n1, D) for dg in digits]
    if any(len(ax) == 0 for ax in axes):
        return []
    grids = np.meshgrid(*axes, indexing="ij")
    C = np.stack([g.ravel() for g in grids], axis=1)              # (nb, d) centres
    lo = np.maximum(C - w, 0)
    hi = np.minimum(C + w, n1 - 1)
    ln = hi - lo + 1
    groups = {}
    for i, key in enumerate(map(tuple, ln)):
        groups.setdefault(key, []).append(i)
    return [(lo[np.array(ix)], np.array(key)) for key, ix in groups.items()]


def _block_indices(lo, ln, n1, d):
    """(nb, k) global indices of the windows, local order x fastest (as ``schwarz.block_of``)."""
    loc = np.meshgrid(*[np.arange(ln[a]) for a in reversed(range(d))], indexing="ij")
    loc = [g.ravel() for g in reversed(loc)]                      # loc[a]: local coordinate on axis a
    idx = np.zeros((lo.shape[0], len(loc[0])), dtype=np.int64)
    for a in range(d):
        idx += (lo[:, a:a + 1] + loc[a][None, :]) * n1 ** a
    return idx


def _block_matrices(Kd, Md, lo, ln, d):
    """A^B = V_B A V_B^T for every block of the group, from A = Σ_a ⊗_b X_b:
    A^B = Σ_a ⊗_b X_b[B_b, B_b] (local order x fastest -> the x factor is the innermost kron)."""
    nb = lo.shape[0]
    sub = {}
    for a in range(d):
        r = lo[:, a:a + 1] + np.arange(ln[a])[None, :]           # (nb, len_a)
        sub[("K", a)] = Kd[r[:, :, None], r[:, None, :]]
        sub[("M", a)] = Md[r[:, :, None], r[:, None, :]]
    k = int(np.prod(ln))
    AB = np.zeros((nb, k, k))
    for a in range(d):
        # kron over axes, slowest (d-1) first: T = X_{d-1} ⊗ ... ⊗ X_0
        T = None
        for b in reversed(range(d)):
            X = sub[("K" if b == a else "M", b)]
            T = X if T is None else (T[:, :, None, :, None] * X[:, None, :, None, :]).reshape(
                nb, T.shape[1] * X.shape[1], -1)
        AB += T
    return AB


class KronTwoLevel:
    """Algorithm 1, multicolour Schwarz order, matrix-free (see module docstring)."""

    def __init__(self, d, p, q, m, s, coarse="vcycle", h_factor=2, coarsest_m=8, cache_bytes=6e9, mg=None):
        self.d, self.p, self.q, self.m, self.s = d, p, q, m, s
        self.n1 = m + p - 2
        self.N = self.n1 ** d
        self.D = s + p
        self.A = KronOperator(p, m, d)
        self.mc = m // h_factor
        R1 = degree_restriction_1d(p, q, m)
        if h_factor == 2:
            R1 = mesh_prolongation_1d(q, m // 2).T @ R1
        self.R1 = sp.csr_matrix(R1)
        self.R1T = sp.csr_matrix(R1.T)
        self.nc1 = R1.shape[0]
        self.Nc = self.nc1 ** d
        if coarse == "vcycle":          # (a QHierarchy of the same (q, m_c, d) may be shared: it is read-only)
            self.mg = mg if mg is not None else QHierarchy(q, self.mc, d, coarsest_m)
            self._csolve = self.mg.vcycle
        elif coarse == "exact":
            self._csolve = spla.factorized(stiffness(q, self.mc, d).tocsc())
        else:
            raise ValueError(coarse)
        self.groups = [_colour_groups(self.n1, d, s, self.D, c) for c in range(self.D ** d)]
        # block inverses are kept between sweeps while they fit (setup-like, not part of the method)
        k = s ** d
        self.keep = self.N * k * k * 8 <= cache_bytes
        self._inv = {}

    def restrict(self, v):
        return kron_apply([self.R1] * self.d, v, self.n1, self.d)

    def prolong(self, e):
        return kron_apply([self.R1T] * self.d, e, self.nc1, self.d)

    def colour_step(self, x, b, colour):
        r = b - self.A.apply(x)                                   # V_B (b - A x) for every block of the colour
        for g, (lo, ln) in enumerate(self.groups[colour]):
            idx = _block_indices(lo, ln, self.n1, self.d)
            if self.keep:
                inv = self._inv.get((colour, g))
                if inv is None:
                    inv = np.linalg.inv(_block_matrices(self.A.Kd, self.A.Md, lo, ln, self.d))
                    self._inv[(colour, g)] = inv
                x[idx] += np.matmul(inv, r[idx][:, :, None])[:, :, 0]
            else:
                AB = _block_matrices(self.A.Kd, self.A.Md, lo, ln, self.d)
                x[idx] += np.linalg.solve(AB, r[idx][:, :, None])[:, :, 0]
        return x

    def sweep(self, x, b):
        for c in range(self.D ** self.d):
            self.colour_step(x, b, c)
        return x

    def iterate(self, x, b):
        self.sweep(x, b)                                          # u^1 = u^0 + S_p(b - A_p u^0)
        dq = self.restrict(b - self.A.apply(x))                   # d_q = I_p^q (b - A_p u^1)
        x += self.prolong(self._csolve(dq))                       # u^1 += I_q^p A_q^{-1} d_q
        return x

    def rate(self, x0, iters=25, last=10):
        """Asymptotic factor, same protocol as ``TwoLevel.rate`` (b = 0, renormalised)."""
        b = np.zeros(self.N)
        x = x0.copy()
        x /= np.linalg.norm(self.A.apply(x))
        ratios = []
        for _ in range(iters):
            self.iterate(x, b)
            rn = np.linalg.norm(self.A.apply(x))
            ratios.append(rn)
            x /= rn
        rt = np.array(ratios[-last:])
        return float(np.exp(np.mean(np.log(rt)))), np.array(ratios)
