"""Pins for oracle/kron.py (the matrix-free Algorithm 1 used for full-size GPU parity) and for
oracle/sampled.py (single rows / single blocks): both against the ASSEMBLED operator
(``assembly.stiffness``, element by element) and the sequential ``TwoLevel`` / ``Schwarz``."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle.assembly import stiffness
from oracle.kron import KronOperator, KronTwoLevel, _block_indices, _block_matrices, _colour_groups
from oracle.sampled import RowOracle
from oracle.schwarz import block_of
from oracle.transfer import restriction
from oracle.twolevel import TwoLevel
from synthetic_inputs import initial_guess, random_rhs


@pytest.mark.parametrize("d,p,m", [(2, 3, 10), (2, 8, 12), (3, 2, 5), (3, 5, 4)])
def test_kron_operator_equals_assembled(d, p, m):
    A = stiffness(p, m, d, method="element")
    x = initial_guess(A.shape[0])
    ref = A @ x
    assert np.abs(KronOperator(p, m, d).apply(x) - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("d,p,m,s", [(2, 3, 9, 3), (2, 5, 8, 5), (3, 3, 5, 3)])
def test_block_matrices_equal_assembled_blocks(d, p, m, s):
    """Every block of every colour: indices == schwarz.block_of, A^B == A[B, B]."""
    A = stiffness(p, m, d, method="element").toarray()
    n1, D, w = m + p - 2, s + p, (s - 1) // 2
    seen = np.zeros(n1 ** d, int)
    op = KronOperator(p, m, d)
    for c in range(D ** d):
        for lo, ln in _colour_groups(n1, d, s, D, c):
            idx = _block_indices(lo, ln, n1, d)
            AB = _block_matrices(op.Kd, op.Md, lo, ln, d)
            for k in range(idx.shape[0]):
                centre = tuple(int(lo[k, a] + (w if lo[k, a] > 0 else ln[a] - 1 - w)) for a in range(d))
                B = idx[k]
                assert np.array_equal(B, block_of(centre, n1, w))
                assert np.abs(AB[k] - A[np.ix_(B, B)]).max() <= 1e-14 * np.abs(A).max()
                seen[B] += 1
    assert seen.min() >= 1


@pytest.mark.parametrize("d,p,q,m,s,coarse,hf", [(2, 3, 1, 24, 3, "vcycle", 2), (2, 5, 2, 16, 5, "exact", 1),
                                                 (3, 3, 1, 8, 3, "vcycle", 2), (2, 8, 2, 16, 7, "vcycle", 2)])
def test_kron_twolevel_equals_twolevel(d, p, q, m, s, coarse, hf):
    """Two iterations of the matrix-free oracle == the assembled sequential oracle (multicolour order)."""
    kt = KronTwoLevel(d, p, q, m, s, coarse, hf)
    tl = TwoLevel(d, p, q, m, s=s, coarse=coarse, h_factor=hf, order="multicolour")
    b, x0 = random_rhs(kt.N), initial_guess(kt.N)
    x1, x2 = x0.copy(), x0.copy()
    for _ in range(2):
        kt.iterate(x1, b)
        tl.iterate(x2, b)
    # the two differ only in rounding: per-block Cholesky vs LU, operator sum order (κ(A_B) <= 4.3e3)
    assert np.linalg.norm(x1 - x2) <= 1e-11 * np.linalg.norm(x2)
    # transfers: 1D factors applied axis by axis == the sparse Kronecker R
    R = restriction(p, q, m, d, hf)
    v = random_rhs(kt.N, seed=5)
    assert np.abs(kt.restrict(v) - R @ v).max() <= 1e-14 * np.abs(R @ v).max()
    e = random_rhs(kt.Nc, seed=6)
    assert np.abs(kt.prolong(e) - R.T @ e).max() <= 1e-14 * np.abs(R.T @ e).max()


def test_kron_inverse_cache_equals_solve():
    """Cached block inverses (reused between sweeps) == fresh dense solves, to rounding."""
    a = KronTwoLevel(2, 4, 1, 32, 3)
    c = KronTwoLevel(2, 4, 1, 32, 3, cache_bytes=0)
    assert a.keep and not c.keep
    b, x0 = random_rhs(a.N), initial_guess(a.N)
    x1, x2 = x0.copy(), x0.copy()
    for _ in range(2):
        a.iterate(x1, b)
        c.iterate(x2, b)
    assert np.linalg.norm(x1 - x2) <= 1e-13 * np.linalg.norm(x2)


@pytest.mark.parametrize("d,p,m,s", [(2, 8, 20, 7), (3, 5, 8, 5)])
def test_row_oracle_equals_assembled(d, p, m, s):
    """sampled.RowOracle (the reference of the sampled full-size checks): apply_rows == rows of the
    element-by-element stiffness; block_update == a dense solve with A[B, B]."""
    A = stiffness(p, m, d, method="element").tocsr()
    ro = RowOracle(p, m, d)
    N, n1, w = A.shape[0], m + p - 2, (s - 1) // 2
    x, b = initial_guess(N), random_rhs(N)
    rows = np.concatenate([[0, N - 1, n1 - 1, n1 * (n1 // 2) + n1 // 2], np.random.default_rng(3).integers(0, N, 30)])
    ref = A[rows] @ x
    assert np.abs(ro.apply_rows(x, rows) - ref).max() <= 1e-14 * np.abs(A).max() * np.abs(x).max() * 10
    Ad = A.toarray()
    for centre in [(0,) * d, (n1 // 2,) * d, (n1 - 1,) + (1,) * (d - 1), (w,) * d]:
        B, dB = ro.block_update(x, b, centre, s)
        assert np.array_equal(B, block_of(centre, n1, w))
        ref = np.linalg.solve(Ad[np.ix_(B, B)], b[B] - Ad[B] @ x)
        # two solves of the same SPD block: agree to ~κ(A_B) eps (κ <= 4.3e3)
        assert np.abs(dB - ref).max() <= 1e-12 * np.abs(ref).max()
