"""ORACLE (test infrastructure only) — Algorithm 1 and the solve loop.

One iteration u^0 -> u^1 (ν1 = 1, ν2 = 0, reading A14):
    u^1 = u^0 + S_p(b - A_p u^0)        one multiplicative Schwarz sweep
    d_p = b - A_p u^1                   defect
    d_q = I_p^q d_p                     restriction
    A_q e_q = d_q                       exact, or one V(1,1) cycle
    u^1 = u^1 + I_q^p e_q               prolongation
Coarse level: q at h (Algorithm 1) or at H = 2h (aggressive); reading A1 gives the
per-config choice.  Solve: stop when ‖b - A x_k‖₂ ≤ rtol ‖b - A x_0‖₂ (A15).
Rate: b = 0, random x_0, renormalise each iteration, geometric mean of the last 10 residual
ratios ("zero right-hand side and a random initial guess").
"""
import numpy as np
import scipy.linalg as sla
import scipy.sparse.linalg as spla

from .assembly import stiffness
from .multigrid import QHierarchy
from .schwarz import Schwarz
from .transfer import restriction


def paper_block_size(p):
    """Block side by degree: 3×3 for p ≤ 4, 5×5 for p = 5, 6, 7×7 for p = 7, 8."""
    if p <= 4:
        return 3
    if p <= 6:
        return 5
    return 7


class TwoLevel:
    def __init__(self, d, p, q, m, s=None, coarse="vcycle", h_factor=2, order="multicolour",
                 coarsest_m=8, A=None):
        self.d, self.p, self.q, self.m = d, p, q, m
        self.s = paper_block_size(p) if s is None else s
        self.n1 = m + p - 2
        self.N = self.n1 ** d
        self.A = (stiffness(p, m, d) if A is None else A).tocsr()
        self.smoother = Schwarz(self.A, self.n1, d, self.s, p, order)
        self.h_factor = h_factor
        self.mc = m // h_factor
        self.R = restriction(p, q, m, d, h_factor).tocsr()
        self.RT = self.R.T.tocsr()
        self.coarse = coarse
        if coarse == "exact":
            Aq = stiffness(q, self.mc, d)
            self.Aq = Aq
            if Aq.shape[0] <= 4096:
                self._csolve = lambda r, f=sla.cho_factor(Aq.toarray(), lower=True): sla.cho_solve(f, r)
            else:
                lu = spla.splu(Aq.tocsc())
                self._csolve = lu.solve
        elif coarse == "vcycle":
            self.mg = QHierarchy(q, self.mc, d, coarsest_m)
            self._csolve = self.mg.vcycle
        else:
            raise ValueError(coarse)

    def residual(self, x, b):
        return b - self.A @ x

    def iterate(self, x, b):
        """One two-level iteration (Algorithm 1), in place; returns x."""
        self.smoother.sweep(x, b)                  # u^1 = u^0 + S_p(b - A_p u^0)
        dp = b - self.A @ x                        # d_p
        dq = self.R @ dp                           # d_q = I_p^q d_p
        eq = self._csolve(dq)                      # A_q e_q = d_q (exact or one V(1,1))
        x += self.RT @ eq                          # u^1 += I_q^p e_q
        return x

    def solve(self, b, x0, rtol=1e-8, maxit=200):
        x = x0.copy()
        r0 = np.linalg.norm(self.residual(x, b))
        hist = [r0]
        it = 0
        while it < maxit and hist[-1] > rtol * r0:
            self.iterate(x, b)
            it += 1
            hist.append(np.linalg.norm(self.residual(x, b)))
        return x, it, np.array(hist)

    def rate(self, x0, iters=30, last=10):
        """Asymptotic factor: b = 0, renormalised residual ratios, geometric mean of the last ``last``."""
        b = np.zeros(self.N)
        x = x0.copy()
        r = np.linalg.norm(self.A @ x)
        x /= r
        ratios = []
        for _ in range(iters):
            self.iterate(x, b)
            rn = np.linalg.norm(self.A @ x)
            ratios.append(rn)
            x /= rn
        rt = np.array(ratios[-last:])
        return float(np.exp(np.mean(np.log(rt)))), np.array(ratios)

    def error_operator(self):
        """Dense two-level error propagation E = (I - P A_q^{-1} R A) S, columns by
        applying one iteration with b = 0 to the unit vectors (small N only)."""
        N = self.N
        E = np.zeros((N, N))
        b = np.zeros(N)
        for j in range(N):
            e = np.zeros(N)
            e[j] = 1.0
            E[:, j] = self.iterate(e, b)
        return E
