"""CPU-only tests of the C-ABI library: it loads, exports every symbol include/iga2l.h declares,
its host-side setup (L0) agrees with the oracle, and it reports errors (no GPU here)."""
import ctypes

import numpy as np
import pytest

import paper_2009_01499_b200 as pkg
from oracle.assembly import matrices_1d
from oracle.transfer import degree_restriction_1d, mesh_prolongation_1d


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()


def test_exports_every_header_symbol():
    L = pkg.lib()
    syms = pkg.header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert b"iga2l" in L.iga2l_version()


def _dense_from_band(B, p):
    n1 = B.shape[0]
    D = np.zeros((n1, n1))
    for i in range(n1):
        for t in range(-p, p + 1):
            if 0 <= i + t < n1:
                D[i, i + t] = B[i, t + p]
    return D


@pytest.mark.parametrize("p,m", [(1, 4), (2, 5), (3, 7), (5, 16), (8, 24), (8, 9)])
def test_host_band_tables_match_oracle(p, m):
    K, M = pkg.host_band_tables(p, m)
    Ko, Mo = matrices_1d(p, m)
    assert np.abs(_dense_from_band(K, p) - Ko).max() <= 1e-14 * np.abs(Ko).max()
    assert np.abs(_dense_from_band(M, p) - Mo).max() <= 1e-14 * np.abs(Mo).max()
    # entries pointing outside the constrained range are exactly zero
    assert np.all(K[0, :p] == 0) and np.all(M[-1, p + 1:] == 0)


@pytest.mark.parametrize("p,q,m,hf", [(2, 1, 16, 1), (3, 1, 8, 1), (3, 1, 16, 2), (5, 2, 16, 2), (8, 2, 32, 2), (4, 2, 12, 2)])
def test_host_restriction_matches_oracle(p, q, m, hf):
    R = pkg.host_restriction_1d(p, q, m, hf)
    Ro = degree_restriction_1d(p, q, m)
    if hf == 2:
        Ro = mesh_prolongation_1d(q, m // 2).T @ Ro
    assert R.shape == Ro.shape
    assert np.abs(R - Ro).max() <= 1e-14 * np.abs(Ro).max()


def test_setup_errors_without_gpu_or_bad_params():
    h = ctypes.c_void_p()
    L = pkg.lib()
    # bad parameters are rejected before any device work, naming the field
    for args, word in [((4, 2, 1, 16, 3, 2), "dim"), ((2, 9, 1, 16, 3, 2), "p"), ((2, 3, 3, 16, 3, 2), "q"),
                       ((2, 3, 1, 16, 4, 3), "block"), ((2, 3, 1, 16, 3, 1), "overlap"),
                       ((2, 3, 1, 15, 3, 2), "n even")]:
        rc = L.iga2l_setup(*args, ctypes.byref(h))
        assert rc == pkg.EPARAM, (args, rc)
        assert word in L.iga2l_last_error().decode()
    import torch
    if not torch.cuda.is_available():
        rc = L.iga2l_setup(2, 2, 1, 16, 3, 2, ctypes.byref(h))
        assert rc == pkg.ECUDA and b"no CUDA device" in L.iga2l_last_error()
        with pytest.raises(pkg.IgaError):
            pkg.Context(2, 2, 1, 16, 3)


@pytest.mark.parametrize("q,m", [(1, 8), (1, 64), (2, 16), (2, 130)])
def test_host_coarse_fd_diagonalises_the_oracle_matrices(q, m):
    """The exact second-level solve's eigen-decomposition against the oracle's own
    1D matrices: V^T M V = I, V^T K V = diag(lam), and the Kronecker inverse equals a sparse solve."""
    import numpy as np
    import scipy.sparse.linalg as spla
    from oracle.assembly import matrices_1d, stiffness
    V, lam = pkg.host_coarse_fd(q, m)
    K, M = matrices_1d(q, m)
    K, M = K.toarray() if hasattr(K, "toarray") else K, M.toarray() if hasattr(M, "toarray") else M
    n = V.shape[0]
    assert np.abs(V.T @ M @ V - np.eye(n)).max() <= 1e-12
    assert np.abs(V.T @ K @ V - np.diag(lam)).max() <= 1e-11 * lam.max()
    # 2D: A^{-1} d = V [(V^T D V) / (lam_j + lam_k)] V^T  (D[y][x])
    d = np.random.default_rng(3).uniform(-1, 1, n * n)
    D = d.reshape(n, n)
    E = V @ ((V.T @ D @ V) / (lam[:, None] + lam[None, :])) @ V.T
    A = stiffness(q, m, 2).tocsc()
    ref = spla.spsolve(A, d)
    assert np.abs(E.ravel() - ref).max() <= 1e-11 * np.abs(ref).max()


@pytest.mark.parametrize("q,n", [(1, 7), (1, 24), (2, 12), (2, 30)])
def test_host_periodic_fd_diagonalises_the_circulant_pencil(q, n):
    """The torus LFA run's exact second level (iga2l_host_periodic_fd): against the oracle's convolution
    stencils (oracle.lfa.stencils_1d, h = 1; the library's tables carry another h, so both are compared up to
    one scale): V diagonalises the circulant pencil (V^T M V ∝ I, V^T K V ∝ diag(λ)); the spectrum equals
    the closed form k̂(θ_j)/m̂(θ_j), θ_j = 2πj/n (circulant symbols); exactly one λ is 0, with a constant
    eigenvector."""
    import numpy as np
    from oracle.lfa import stencils_1d
    V, lam = pkg.host_periodic_fd(q, n)
    _, _, kq, mq, _ = stencils_1d(q, q)
    K, M = np.zeros((n, n)), np.zeros((n, n))
    for i in range(n):
        for d, v in kq.items():
            K[i, (i + d) % n] += v
        for d, v in mq.items():
            M[i, (i + d) % n] += v
    VMV, VKV = V.T @ M @ V, V.T @ K @ V
    c = VMV[0, 0]
    assert np.abs(VMV - c * np.eye(n)).max() <= 1e-12 * c
    assert np.abs(VKV - np.diag(np.diag(VKV))).max() <= 1e-11 * np.abs(VKV).max()
    assert np.sum(lam == 0.0) == 1
    nz = lam != 0.0
    ratio = np.diag(VKV)[nz] / lam[nz]
    assert np.abs(ratio / ratio[0] - 1).max() <= 1e-11
    th = 2 * np.pi * np.arange(n) / n
    khat = sum(v * np.cos(d * th) for d, v in kq.items())
    mhat = sum(v * np.cos(d * th) for d, v in mq.items())
    closed = np.sort(khat / mhat)
    got = np.sort(lam)
    assert abs(closed[0]) <= 1e-13 and got[0] == 0.0
    assert np.abs(got[1:] / got[-1] - closed[1:] / closed[-1]).max() <= 1e-12
    j0 = int(np.argmin(np.abs(lam)))
    v0 = V[:, j0]
    assert np.abs(v0 - v0.mean()).max() <= 1e-12 * np.abs(v0).max()


# ---- quarter annulus: the library's host setup against the oracle's 2D assembly ----
def _dense_band(B, p):
    n1, W = B.shape
    D = np.zeros((n1, n1))
    for i in range(n1):
        for t in range(W):
            j = i + t - p
            if 0 <= j < n1:
                D[i, j] = B[i, t]
    return D


@pytest.mark.parametrize("p,m", [(2, 4), (3, 6), (5, 8), (8, 12)])
def test_host_annulus_tables_give_the_assembled_operator(p, m):
    """My ⊗ Kx + Ky ⊗ Mx from the library's per-axis tables equals the oracle's element-by-element 2D
    stiffness on the exact geometry (NURBS weights from the blossom here, L2 projection there)."""
    from oracle import annulus as an
    Kx, Mx, Ky, My = (_dense_band(T, p) for T in pkg.host_annulus_tables(p, m))
    A = an.assemble(p, m)["A"].toarray()
    assert np.abs(np.kron(My, Kx) + np.kron(Ky, Mx) - A).max() <= 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("p,m,hf", [(3, 8, 2), (5, 8, 1), (4, 12, 2)])
def test_host_annulus_restriction_matches_oracle(p, m, hf):
    """Ry ⊗ Rx (per-axis lumped L2 restriction, composed with the NURBS / B-spline embedding) equals the
    oracle's 2D R = P^T D^{-1} C."""
    import scipy.sparse as sp
    from oracle import annulus as an
    Rx = pkg.host_annulus_restriction_1d(0, p, 2, m, hf)
    Ry = pkg.host_annulus_restriction_1d(1, p, 2, m, hf)
    C = an.assemble(p, m, q=2, want=("C",))["C"]
    R = sp.diags(1.0 / an.lumped_q_mass(2, m)) @ C
    if hf == 2:
        R = an.embedding(2, m // 2).T @ R
    R = R.toarray()
    assert np.abs(np.kron(Ry, Rx) - R).max() <= 1e-13 * np.abs(R).max()


def test_host_annulus_load_matches_oracle():
    from oracle import annulus as an
    b = pkg.host_annulus_load(3, 8)
    ref = an.assemble(3, 8, want=("b",))["b"]
    assert np.abs(b - ref).max() <= 1e-13 * np.abs(ref).max()
