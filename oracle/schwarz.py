"""ORACLE (test infrastructure only) — overlapping multiplicative Schwarz.

One block per grid point ("maximum overlapping ... every block is related to a grid-point,
involving that grid-point and its neighbors"); in d dimensions the block of centre c is
the s^d window ∏_a [c_a - w, c_a + w] (w = (s-1)/2), clipped to the grid (reading A3, no
ghost unknowns).  A block step is

    x <- x + V_B^T (A^{B})^{-1} V_B (b - A x),      A^{B} = V_B A V_B^T,

applied block after block ("multiplicative"), each step seeing the x left by the previous one.

Orders (reading A4/A5):
  * ``lex``         — centres in ascending flattened index (x fastest).
  * ``multicolour`` — colour(c) = Σ_a (c_a mod D) D^a with D = s + p, colours ascending, lex
                      inside a colour.  Same-colour blocks are ≥ p+1 apart on some axis, so
                      A[B1, B2] = 0 and the blocks are disjoint: this equals a parallel colour
                      step (pinned in tests), which is what the GPU runs.
The paper's own "three-colour" pattern is defined in [nuestropaper2018], not in the container.
"""
import numpy as np
import scipy.linalg as sla


def block_of(centre, n1, w):
    """Global (x-fastest) indices of the clipped window around ``centre`` (tuple, axis 0 = x)."""
    d = len(centre)
    rng = [np.arange(max(0, c - w), min(n1 - 1, c + w) + 1) for c in centre]
    # axis a contributes i_a * n1^a; meshgrid over reversed axes + C-order ravel gives x fastest
    grids = np.meshgrid(*[rng[a] for a in reversed(range(d))], indexing="ij")
    flat = np.zeros(grids[0].shape, dtype=np.int64)
    for k, a in enumerate(reversed(range(d))):
        flat += grids[k] * n1 ** a
    return flat.ravel()


def centres(n1, d):
    """All centres as tuples (x, y[, z]) in ascending flattened index."""
    out = []
    for g in range(n1 ** d):
        out.append(tuple((g // n1 ** a) % n1 for a in range(d)))
    return out


def colour_of(centre, D):
    """Reading A5: c = Σ_a (i_a mod D) D^a (axis 0 = x)."""
    return sum((c % D) * D ** a for a, c in enumerate(centre))


def ordered_centres(n1, d, s, p, order):
    cs = centres(n1, d)
    if order == "lex":
        return cs
    if order == "multicolour":
        D = s + p
        return sorted(cs, key=lambda c: (colour_of(c, D), sum(ci * n1 ** a for a, ci in enumerate(c))))
    raise ValueError(order)


class Schwarz:
    """Multiplicative Schwarz smoother S_p with dense Cholesky local solves."""

    def __init__(self, A, n1, d, s, p, order="multicolour"):
        if s % 2 != 1:
            raise ValueError("block side s must be odd")
        self.A = A.tocsr()
        self.n1, self.d, self.s, self.p, self.w = n1, d, s, p, (s - 1) // 2
        self.order = order
        self.seq = ordered_centres(n1, d, s, p, order)
        self._fac = {}
        k = s ** d
        # per-block (rows, factor) cache (setup-like, not part of the method), bounded in memory
        self.cache = n1 ** d * k * min(2 * p + 1, n1) ** d <= 3e7

    def _factor(self, c):
        f = self._fac.get(c)
        if f is None:
            B = block_of(c, self.n1, self.w)
            rows = self.A[B]                                   # V_B A
            AB = rows[:, B].toarray()                          # A^{B} = V_B A V_B^T
            f = (B, sla.cho_factor(AB, lower=True), rows)
            if self.cache:
                self._fac[c] = f
        return f

    def step(self, x, b, c):
        """One block step for centre c (in place)."""
        B, fac, rows = self._factor(c)
        r = b[B] - rows @ x                                    # V_B (b - A x)
        x[B] += sla.cho_solve(fac, r, check_finite=False)                        # V_B^T (A^B)^{-1} (...)

    def sweep(self, x, b, centres_subset=None):
        """One multiplicative sweep over all blocks in the chosen order (in place, returns x)."""
        for c in (self.seq if centres_subset is None else centres_subset):
            self.step(x, b, c)
        return x

    def colour_step_parallel(self, x, b, colour):
        """All blocks of one colour computed from the SAME x, then applied (the GPU's formulation).
        Equal to the sequential colour step because same-colour blocks are A-decoupled (A4);
        the equality is pinned in tests, this function is only used to check it."""
        D = self.s + self.p
        x0 = x.copy()
        upd = []
        for c in self.seq:
            if colour_of(c, D) != colour:
                continue
            B, fac, rows = self._factor(c)
            upd.append((B, sla.cho_solve(fac, b[B] - rows @ x0, check_finite=False)))
        for B, dB in upd:
            x[B] += dB
        return x
