"""Seeded synthetic inputs and workload shapes, shared by the oracle tests, the GPU tests and
bench.py.  This module holds NONE of the method's arithmetic (no basis, quadrature, operator,
transfer or smoother): only random vectors and the BASELINE.json configuration shapes.

Reading A16: the random initial guess is U[-1, 1] from seed 0, drawn once on the
host with ``numpy.random.default_rng(seed).uniform(-1, 1, N)`` in the x-fastest layout and handed
unchanged to both the oracle and the GPU path.
"""
import numpy as np

# BASELINE.json configs.  coarse: "exact" (dense, same h) or "vcycle"
# (one V(1,1), aggressive H = 2h).  s = paper block side.
CONFIGS = {
    "C1": dict(d=2, p=2, q=1, m=16, s=3, coarse="exact", h_factor=1),
    "C2p3": dict(d=2, p=3, q=1, m=256, s=3, coarse="vcycle", h_factor=2),
    "C2p4": dict(d=2, p=4, q=1, m=256, s=3, coarse="vcycle", h_factor=2),
    "C2p5": dict(d=2, p=5, q=1, m=256, s=5, coarse="vcycle", h_factor=2),
    "C3": dict(d=2, p=8, q=2, m=1024, s=7, coarse="vcycle", h_factor=2),
    "C4": dict(d=3, p=3, q=1, m=128, s=3, coarse="vcycle", h_factor=2),
    "C5": dict(d=3, p=5, q=2, m=256, s=5, coarse="vcycle", h_factor=2),
}


def n_dofs(cfg):
    return (cfg["m"] + cfg["p"] - 2) ** cfg["d"]


def initial_guess(N, seed=0):
    """x_0 ~ U[-1, 1] ("random vector"; A16)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, N)


def random_rhs(N, seed=1):
    """An arbitrary right-hand side b ~ U[-1, 1] for parity runs (any b is a valid solver input)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, N)
