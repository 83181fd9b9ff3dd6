"""ORACLE (test infrastructure only) — the q-level h-multigrid V(1,1) cycle.

"we apply one V(1,1)-cycle that uses a red-black Gauss-Seidel iteration as smoother".
Readings: A10 — the operator on every level is the rediscretized A_q; A8 — the mesh
transfers are the exact knot-insertion embedding P and its unscaled transpose; A11 — red-black
is not a decoupled colouring for the (2q+1)^d-point IGA stencils, so the smoother is the
(q+1)^d-colour Gauss–Seidel, colour(c) = Σ_a (c_a mod (q+1)) (q+1)^a, colours ascending
(an exact Gauss–Seidel sweep in colour-major order); A12 — coarsen until m ≤ 8,
direct solve there; A13 — zero initial guess on the coarse level, one cycle.
"""
import numpy as np
import scipy.linalg as sla

from .assembly import stiffness
from .transfer import mesh_prolongation


def _colour_sets(n, d, ncol_axis):
    idx = np.arange(n ** d)
    col = np.zeros(n ** d, dtype=np.int64)
    for a in range(d):
        col += ((idx // n ** a) % n % ncol_axis) * ncol_axis ** a
    return [idx[col == c] for c in range(ncol_axis ** d)]


class QHierarchy:
    def __init__(self, q, m0, d, coarsest_m=8):
        self.q, self.d = q, d
        self.levels = []
        m = m0
        while True:
            A = stiffness(q, m, d).tocsr()
            n = m + q - 2
            lev = {"m": m, "n": n, "A": A, "diag": A.diagonal().copy(),
                   "colours": _colour_sets(n, d, q + 1)}
            self.levels.append(lev)
            if m <= coarsest_m:
                lev["chol"] = sla.cho_factor(A.toarray(), lower=True)
                break
            if m % 2:
                raise ValueError(f"V-cycle needs m divisible by 2 down to <= {coarsest_m}; got m={m}")
            lev["P"] = mesh_prolongation(q, m // 2, d)
            m //= 2

    def gs(self, l, x, b):
        """One (q+1)^d-colour Gauss–Seidel sweep; within a colour the points are decoupled
        (pinned equal to the pointwise sequential sweep in tests), so each colour is one update
        x_i += (b_i - (A x)_i) / A_ii."""
        lev = self.levels[l]
        A, dg = lev["A"], lev["diag"]
        for pts in lev["colours"]:
            x[pts] += (b[pts] - A[pts] @ x) / dg[pts]
        return x

    def gs_pointwise(self, l, x, b):
        """Sequential pointwise Gauss–Seidel in the same colour-major order (for the pin only)."""
        lev = self.levels[l]
        A, dg = lev["A"], lev["diag"]
        for pts in lev["colours"]:
            for i in pts:
                x[i] += (b[i] - A[i].dot(x)[0]) / dg[i]
        return x

    def vcycle(self, b, l=0):
        """One V(1,1) cycle for A_q e = b with zero initial guess."""
        lev = self.levels[l]
        if "chol" in lev:
            return sla.cho_solve(lev["chol"], b)
        x = np.zeros_like(b)
        self.gs(l, x, b)                              # pre-smoothing (ν1 = 1)
        r = b - lev["A"] @ x
        rc = lev["P"].T @ r                           # restriction = P^T (A8)
        ec = self.vcycle(rc, l + 1)
        x += lev["P"] @ ec                            # prolongation
        self.gs(l, x, b)                              # post-smoothing (ν2 = 1)
        return x
