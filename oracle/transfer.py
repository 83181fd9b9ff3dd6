"""ORACLE (test infrastructure only) — inter-level transfers.

Degree transfer at the same h:
    M_q^q u_q = M_p^q u_p,   I_p^q = (M_q^q)^{-1} M_p^q,   I_q^p = (M_p^q)^T (M_q^q)^{-T},
with M_q^q replaced by its row-sum lumping D ("row-sum lumping").  Reading A6: D_ii is
the row sum of the UNCONSTRAINED q-level mass at the constrained rows (= ∫ φ_i^q by partition
of unity).  Reading A7: prolongation = M_c^T D^{-1} = R^T.

Mesh transfer h <-> 2h at fixed degree q ("standard"): reading A8 — the
prolongation is the exact embedding S^q_{2h} ⊂ S^q_h (nested spaces), and restriction is its
plain (unscaled) transpose.  The oracle computes the embedding as the L2 projection
P = M_h^{-1} M_{h,2h}, which is exact because the coarse functions lie in the fine space.

Aggressive coarsening (reading A9): R_ag = P_mesh^T ∘ R_degree, P_ag = R_ag^T.
All d-dim operators are Kronecker products of the 1D factors (tensor-product bases).
"""
import functools

import numpy as np
import scipy.sparse as sp

from .assembly import cross_mass_1d, matrices_1d
from .bspline import basis, knot_vector, span_basis, span_rule


def lumped_mass_1d(q, m):
    """D = row sums of the unconstrained q-level mass M_q^q, kept at constrained rows (A6)."""
    _, Mfull = matrices_1d(q, m, constrained=False)
    return Mfull.sum(axis=1)[1:-1]


def degree_restriction_1d(p, q, m):
    """R1 = D^{-1} M_p^q  (n1_q × n1_p), the lumped L2 projection S_h^p -> S_h^q."""
    D = lumped_mass_1d(q, m)
    Mc = cross_mass_1d(q, p, m)
    return Mc / D[:, None]


def mesh_prolongation_1d(q, m_coarse, constrained=True):
    """Embedding of S^q_{2h} (m_coarse spans) into S^q_h (2 m_coarse spans) (A8):
    P = M_h^{-1} M_{h,2h}, M_{h,2h}[i, j] = ∫ N_i^{q,h} N_j^{q,2h}, integrated span by span on
    the fine mesh with q+1 Gauss points (both factors are degree-q polynomials there)."""
    m_f = 2 * m_coarse
    xf, xc = knot_vector(q, m_f), knot_vector(q, m_coarse)
    _, Mh = matrices_1d(q, m_f, constrained=False)
    Mhc = np.zeros((m_f + q, m_coarse + q))
    for e in range(m_f):
        xs, ws = span_rule(m_f, e, q + 1)
        Nf = np.zeros((len(xs), m_f + q))                  # all functions; only the q+1 on this span
        Nc = np.zeros((len(xs), m_coarse + q))             # (fine) / coarse span e // 2 are non-zero
        Nf[:, e:e + q + 1] = span_basis(xf, q, e, xs)
        Nc[:, e // 2:e // 2 + q + 1] = span_basis(xc, q, e // 2, xs)
        Mhc += Nf.T @ (ws[:, None] * Nc)
    P = np.linalg.solve(Mh, Mhc)
    P[np.abs(P) < 1e-14] = 0.0      # exact zeros outside the support (solve leaves ~1e-17 dust)
    if constrained:
        P = P[1:-1, 1:-1]
    return P


def kron_nd(mats_1d_slowest_first):
    return functools.reduce(lambda u, v: sp.kron(u, v, format="csr"),
                            [sp.csr_matrix(a) for a in mats_1d_slowest_first])


def restriction(p, q, m, d, h_factor):
    """d-dim restriction fine(p, h) -> coarse(q, h_factor*h).
    h_factor = 1: R = ⊗ R1.  h_factor = 2: R = ⊗ (P_m1^T R1) (A9)."""
    R1 = degree_restriction_1d(p, q, m)
    if h_factor == 2:
        if m % 2:
            raise ValueError("aggressive coarsening needs even m")
        R1 = mesh_prolongation_1d(q, m // 2).T @ R1
    elif h_factor != 1:
        raise ValueError("h_factor must be 1 or 2")
    return kron_nd([R1] * d)


def mesh_prolongation(q, m_coarse, d):
    """d-dim embedding S^q_{2h} -> S^q_h (tensor product of the 1D embedding)."""
    return kron_nd([mesh_prolongation_1d(q, m_coarse)] * d)
