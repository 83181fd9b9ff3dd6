"""ORACLE (test infrastructure only) — single rows / single blocks at sizes where the sparse
matrix is too large to assemble (C3-C5 at full size).

Both use the tensor-product identity A_p = Σ_a ⊗_b (K if b == a else M), pinned equal
to the element-by-element assembly in tests/test_oracle_assembly.py, with the oracle's own 1D
matrices.  A block step is the definition of: x_B += (A^B)^{-1} (b - A x)_B with a dense
A^B = V_B A V_B^T (solved with numpy.linalg.solve).
"""
import numpy as np

from .assembly import matrices_1d


class RowOracle:
    def __init__(self, p, m, d):
        self.p, self.m, self.d = p, m, d
        self.n1 = m + p - 2
        self.K, self.M = matrices_1d(p, m)

    def _coords(self, g):
        return [(g // self.n1 ** a) % self.n1 for a in range(self.d)]

    def entry(self, gi, gj):
        ci, cj = self._coords(gi), self._coords(gj)
        v = 0.0
        for a in range(self.d):
            t = 1.0
            for b in range(self.d):
                X = self.K if a == b else self.M
                t *= X[ci[b], cj[b]]
            v += t
        return v

    def row_window(self, g):
        """Column indices and values of row g of A_p (the (2p+1)^d stencil, clipped)."""
        ci = self._coords(g)
        rng = [np.arange(max(0, c - self.p), min(self.n1 - 1, c + self.p) + 1) for c in ci]
        grids = np.meshgrid(*rng, indexing="ij")
        cols = np.zeros(grids[0].shape, dtype=np.int64)
        vals = np.zeros(grids[0].shape)
        for a in range(self.d):
            cols += grids[a] * self.n1 ** a
        for a in range(self.d):
            t = np.ones(grids[0].shape)
            for b in range(self.d):
                X = self.K if a == b else self.M
                t = t * X[ci[b], grids[b]]
            vals += t
        return cols.ravel(), vals.ravel()

    def apply_rows(self, x, rows):
        out = np.empty(len(rows))
        for k, g in enumerate(rows):
            cols, vals = self.row_window(int(g))
            out[k] = vals @ x[cols]
        return out

    def block_update(self, x, b, centre, s):
        """Correction δ_B of the block centred at ``centre`` (tuple, axis 0 = x) for the current x."""
        w = (s - 1) // 2
        rng = [np.arange(max(0, c - w), min(self.n1 - 1, c + w) + 1) for c in centre]
        grids = np.meshgrid(*[rng[a] for a in reversed(range(self.d))], indexing="ij")
        B = np.zeros(grids[0].shape, dtype=np.int64)
        for k, a in enumerate(reversed(range(self.d))):
            B += grids[k] * self.n1 ** a
        B = B.ravel()
        r = b[B] - self.apply_rows(x, B)
        AB = np.array([[self.entry(i, j) for j in B] for i in B])
        return B, np.linalg.solve(AB, r)
