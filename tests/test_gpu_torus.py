"""GPU: the torus LFA run against the oracle's block LFA.

iga2l_lfa_torus power-iterates the two-grid error operator of the multicolour method on an
n x n periodic grid with the library's kernels (padded colour sweeps, residual, periodic transfers,
Kronecker fast-diagonalisation coarse solve).  With n = nk L (L the Bloch cell of the analysis, nk even)
the torus spectrum is exactly the union of the Bloch-cell spectra on the oracle's nk^2 frequency grid, so
the measured spectral radius must equal `oracle.lfa.rho_2g` / `rho_2g_ag` at the same nk (power-iteration
accuracy: 1%); and the measured factor must not depend on the seed.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2009_01499_b200 as pkg  # noqa: E402
from oracle import lfa  # noqa: E402


@pytest.mark.parametrize("p,q,s,nk", [(2, 1, 3, 4), (3, 1, 3, 4), (4, 1, 3, 2), (5, 1, 5, 2), (8, 2, 7, 2)],
                         ids=["p2", "p3", "p4", "p5", "p8q2"])
def test_torus_two_grid_equals_block_lfa(p, q, s, nk):
    """Table 1's setting (exact degree-q level, same h): ρ(torus, n = nk (s + p)) == ρ_2g(nk)."""
    n = nk * (s + p)
    ref = lfa.rho_2g(p, q, s, 2, nk=nk)
    got = pkg.lfa_torus(p, q, n, s, h_factor=1, iters=400, seed=1)
    assert abs(got - ref) <= 0.01 * ref, (got, ref)


@pytest.mark.parametrize("p,q,s,nk", [(3, 1, 3, 2), (4, 1, 3, 2)], ids=["p3", "p4"])
def test_torus_aggressive_equals_block_lfa(p, q, s, nk):
    """Table 3's setting (degree q on H = 2h, exact): ρ(torus, n = nk L) == ρ_2g^ag(nk), L the analysis cell."""
    L = lfa._cell(p, q, s)
    n = nk * L
    ref = lfa.rho_2g_ag(p, q, s, 2, nk=nk)
    got = pkg.lfa_torus(p, q, n, s, h_factor=2, iters=400, seed=2)
    assert abs(got - ref) <= 0.01 * ref, (got, ref)


@pytest.mark.parametrize("p,q,s,nk", [(2, 1, 3, 2), (3, 1, 3, 2), (4, 1, 3, 2), (8, 2, 7, 2)], ids=["p2", "p3", "p4", "p8q2"])
def test_torus_three_grid_equals_block_lfa(p, q, s, nk):
    """Table 2's setting (q-level by one two-grid cycle, (q+1)^2-colour GS, exact 2h): == ρ_3g(nk)."""
    L = lfa._cell(p, q, s)
    n = nk * L
    ref = lfa.rho_3g(p, q, s, 2, nk=nk)
    got = pkg.lfa_torus(p, q, n, s, h_factor=3, iters=400, seed=3)
    assert abs(got - ref) <= 0.01 * ref, (got, ref)


def test_torus_seed_independent_and_errors():
    a = pkg.lfa_torus(3, 1, 24, 3, iters=300, seed=3)
    b = pkg.lfa_torus(3, 1, 24, 3, iters=300, seed=4)
    assert abs(a - b) <= 0.01 * a
    with pytest.raises(pkg.IgaError):
        pkg.lfa_torus(3, 1, 25, 3)                       # n not a multiple of s + p
    with pytest.raises(pkg.IgaError):
        pkg.lfa_torus(3, 1, 24, 3, h_factor=3, dim=3)    # the three-grid run is 2D


@pytest.mark.parametrize("p,s,hf", [(2, 3, 1), (3, 3, 1), (3, 3, 2)], ids=["p2", "p3", "p3_ag"])
def test_torus_3d_equals_block_lfa(p, s, hf):
    """3D (reading A25; no paper value): the torus run == the oracle's 3D block LFA on the nk = 2 grid."""
    L = (s + p) if hf == 1 else lfa._cell(p, 1, s)
    n = 2 * L
    ref = (lfa.rho_2g if hf == 1 else lfa.rho_2g_ag)(p, 1, s, 3, nk=2)
    got = pkg.lfa_torus(p, 1, n, s, h_factor=hf, iters=300, seed=4, dim=3)
    assert abs(got - ref) <= 0.01 * ref, (got, ref)
