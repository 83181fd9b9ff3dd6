"""Pins for oracle/schwarz.py and oracle/multigrid.py: special cases that reduce to textbook
methods (exact solve, Gauss–Seidel), the A-norm contraction of multiplicative Schwarz, the
decoupling of the multicolour order (reading A4) and of the (q+1)^d-colour GS (reading A11)."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import assembly as A
from oracle.multigrid import QHierarchy
from oracle.schwarz import Schwarz, block_of, colour_of, centres


def test_block_clipping_counts():
    # 5x5 grid, 3x3 blocks -> 25 blocks; 9 interior-centred blocks have 9 unknowns, corners 4
    n1 = 5
    sizes = {c: len(block_of(c, n1, 1)) for c in centres(n1, 2)}
    assert len(sizes) == 25
    assert sum(1 for c, k in sizes.items() if 1 <= c[0] <= 3 and 1 <= c[1] <= 3 and k == 9) == 9
    assert sizes[(0, 0)] == sizes[(4, 4)] == sizes[(0, 4)] == 4
    # every unknown lies in >= 1 and <= s^d blocks
    cover = np.zeros(n1 * n1, int)
    for c in sizes:
        cover[block_of(c, n1, 1)] += 1
    assert cover.min() >= 1 and cover.max() <= 9


def _problem(p=3, m=6, d=2, seed=0):
    Ap = A.stiffness(p, m, d)
    N = Ap.shape[0]
    b = np.random.default_rng(seed).uniform(-1, 1, N)
    x = np.random.default_rng(seed + 1).uniform(-1, 1, N)
    return Ap, b, x


def test_whole_grid_block_is_exact_solve():
    # a block covering the whole grid is an exact solve
    p, m = 3, 5
    Ap, b, x = _problem(p, m)
    n1 = m + p - 2
    sm = Schwarz(Ap, n1, 2, s=2 * n1 + 1, p=p, order="lex")
    sm.step(x, b, sm.seq[0])
    assert np.linalg.norm(b - Ap @ x) < 1e-12 * np.linalg.norm(b)


def test_unit_blocks_are_gauss_seidel():
    # 1x1 blocks in lex order = pointwise Gauss–Seidel (written out independently here)
    p, m = 2, 6
    Ap, b, x = _problem(p, m)
    y = x.copy()
    n1 = m + p - 2
    Schwarz(Ap, n1, 2, s=1, p=p, order="lex").sweep(x, b)
    Ad = Ap.toarray()
    for i in range(len(y)):
        y[i] += (b[i] - Ad[i] @ y) / Ad[i, i]
    assert np.allclose(x, y, atol=1e-13)


@pytest.mark.parametrize("order", ["lex", "multicolour"])
def test_a_norm_error_non_increasing(order):
    # each block step is an A-orthogonal projection, so ‖u* - x‖_A never increases
    p, m = 4, 6
    Ap, b, x = _problem(p, m)
    u = spla.spsolve(Ap.tocsc(), b)
    n1 = m + p - 2
    sm = Schwarz(Ap, n1, 2, s=3, p=p, order=order)
    def anorm(v):
        return float(np.sqrt((u - v) @ (Ap @ (u - v))))
    prev = anorm(x)
    for c in sm.seq:
        sm.step(x, b, c)
        cur = anorm(x)
        assert cur <= prev * (1 + 1e-12)
        prev = cur


@pytest.mark.parametrize("d,p,m,s", [(2, 2, 12, 3), (2, 4, 9, 3), (2, 5, 8, 5), (3, 2, 6, 3)])
def test_multicolour_blocks_decoupled_and_parallel_equals_sequential(d, p, m, s):
    Ap, b, x = _problem(p, m, d)
    n1 = m + p - 2
    sm = Schwarz(Ap, n1, d, s=s, p=p, order="multicolour")
    D = s + p
    Ad = Ap.toarray()
    by_col = {}
    for c in sm.seq:
        by_col.setdefault(colour_of(c, D), []).append(c)
    # A[B1, B2] = 0 and B1 ∩ B2 = ∅ for same-colour blocks (reading A4)
    for col, cs in list(by_col.items())[:: max(1, len(by_col) // 7)]:
        for i in range(len(cs)):
            for j in range(i + 1, len(cs)):
                B1, B2 = block_of(cs[i], n1, sm.w), block_of(cs[j], n1, sm.w)
                assert not np.any(Ad[np.ix_(B1, B2)])
    # sequential colour-major sweep == colour-parallel sweep, bitwise
    x_seq = sm.sweep(x.copy(), b)
    x_par = x.copy()
    for col in sorted(by_col):
        sm.colour_step_parallel(x_par, b, col)
    assert np.array_equal(x_seq, x_par)
    # a within-colour permutation gives the bitwise-identical iterate
    rng = np.random.default_rng(5)
    perm = []
    for col in sorted(by_col):
        cs = list(by_col[col])
        rng.shuffle(cs)
        perm += cs
    assert np.array_equal(sm.sweep(x.copy(), b, perm), x_seq)


def test_fixed_point():
    p, m = 3, 7
    Ap, b, _ = _problem(p, m)
    u = spla.spsolve(Ap.tocsc(), b)
    n1 = m + p - 2
    x = Schwarz(Ap, n1, 2, s=3, p=p).sweep(u.copy(), b)
    assert np.linalg.norm(x - u) < 1e-12 * np.linalg.norm(u)


@pytest.mark.parametrize("q,d", [(1, 2), (2, 2), (1, 3)])
def test_colour_gs_equals_pointwise_gs(q, d):
    H = QHierarchy(q, 8, d)
    n = H.levels[0]["n"]
    rng = np.random.default_rng(2)
    b = rng.uniform(-1, 1, n ** d)
    x = rng.uniform(-1, 1, n ** d)
    assert np.allclose(H.gs(0, x.copy(), b), H.gs_pointwise(0, x.copy(), b), atol=1e-14, rtol=0)


@pytest.mark.parametrize("q,m", [(1, 32), (2, 32)])
def test_vcycle_contracts(q, m):
    # one V(1,1) with zero initial guess is a contraction; SURVEY A11 expects 0.035 (q=1), 0.218 (q=2)
    H = QHierarchy(q, m, 2)
    assert [lv["m"] for lv in H.levels] == [32, 16, 8]
    Aq = H.levels[0]["A"]
    b = np.random.default_rng(0).uniform(-1, 1, Aq.shape[0])
    u = spla.spsolve(Aq.tocsc(), b)
    # error propagation of the V-cycle as a solver: e_{k+1} = e_k - V(A e_k)
    x = np.zeros_like(b)
    ratios = []
    for _ in range(5):
        e0 = np.linalg.norm(u - x)
        x = x + H.vcycle(b - Aq @ x)
        ratios.append(np.linalg.norm(u - x) / e0)
    assert max(ratios[1:]) < (0.1 if q == 1 else 0.35), ratios


def test_single_level_hierarchy_is_exact():
    H = QHierarchy(1, 8, 2)
    Aq = H.levels[0]["A"]
    b = np.random.default_rng(0).uniform(-1, 1, Aq.shape[0])
    assert np.linalg.norm(Aq @ H.vcycle(b) - b) < 1e-12
