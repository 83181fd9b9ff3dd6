"""Torus LFA run on the GPU (iga2l_lfa_torus) against the oracle's block LFA on the same frequency grid
(SURVEY §8(f) row 2): two-grid (Table 1's setting) for p = 2..8 with the paper's block sizes, and the
aggressive two-grid (Table 3's) for p = 2..5; nk^2 Bloch frequencies <-> an n = nk L torus.
python tools/lfa_torus_table.py > profiles/lfa_torus_r02.txt"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01499_b200 as pkg  # noqa: E402
from oracle import lfa  # noqa: E402

S = {2: 3, 3: 3, 4: 3, 5: 5, 6: 5, 7: 7, 8: 7}
print("two-grid, exact degree-q level at the same h (Table 1's setting): torus rho vs block LFA rho_2g")
print(f"{'p':>2} {'q':>2} {'s':>2} {'nk':>3} {'n':>4} {'torus':>9} {'LFA':>9} {'rel':>9} {'gpu s':>6}")
for p in range(2, 9):
    for q in ((1, 2) if p == 8 else (1,)):
        s = S[p]
        for nk in (2, 4, 8):
            n = nk * (s + p)
            t0 = time.time()
            got = pkg.lfa_torus(p, q, n, s, h_factor=1, iters=400, seed=1)
            dt = time.time() - t0
            ref = lfa.rho_2g(p, q, s, 2, nk=nk)
            print(f"{p:2d} {q:2d} {s:2d} {nk:3d} {n:4d} {got:9.5f} {ref:9.5f} {abs(got - ref) / ref:9.2e} {dt:6.2f}",
                  flush=True)
print()
print("aggressive two-grid, degree q on H = 2h, exact (Table 3's setting): torus rho vs block LFA rho_2g^ag")
for p in range(2, 6):
    s, q = S[p], 1
    L = lfa._cell(p, q, s)
    for nk in (2, 4):
        n = nk * L
        t0 = time.time()
        got = pkg.lfa_torus(p, q, n, s, h_factor=2, iters=400, seed=2)
        dt = time.time() - t0
        ref = lfa.rho_2g_ag(p, q, s, 2, nk=nk)
        print(f"{p:2d} {q:2d} {s:2d} {nk:3d} {n:4d} {got:9.5f} {ref:9.5f} {abs(got - ref) / ref:9.2e} {dt:6.2f}",
              flush=True)
print()
print("three-grid, q-level by one two-grid cycle (Table 2's setting): torus rho vs block LFA rho_3g")
for p in (2, 3, 4, 5, 8):
    s, q = S[p], (2 if p == 8 else 1)
    L = lfa._cell(p, q, s)
    for nk in (2,):
        n = nk * L
        t0 = time.time()
        got = pkg.lfa_torus(p, q, n, s, h_factor=3, iters=400, seed=2)
        dt = time.time() - t0
        ref = lfa.rho_3g(p, q, s, 2, nk=nk)
        print(f"{p:2d} {q:2d} {s:2d} {nk:3d} {n:4d} {got:9.5f} {ref:9.5f} {abs(got - ref) / ref:9.2e} {dt:6.2f}",
              flush=True)
print()
print("3D (reading A25, no paper values): torus vs the oracle's 3D block LFA, nk = 2")
for p, s, hf in ((2, 3, 1), (3, 3, 1), (3, 3, 2), (4, 3, 1)):
    L = (s + p) if hf == 1 else lfa._cell(p, 1, s)
    n = 2 * L
    t0 = time.time()
    got = pkg.lfa_torus(p, 1, n, s, h_factor=hf, iters=300, seed=4, dim=3)
    dt = time.time() - t0
    ref = (lfa.rho_2g if hf == 1 else lfa.rho_2g_ag)(p, 1, s, 3, nk=2)
    print(f"{p:2d}  1 {s:2d}   2 {n:4d} {got:9.5f} {ref:9.5f} {abs(got - ref) / ref:9.2e} {dt:6.2f}  (h_factor {hf})",
          flush=True)
print("3D predictions beyond the oracle's reach (torus only): C4's and C5's (p, s), aggressive 2h like the configs")
for p, s, q, nk in ((3, 3, 1, 4), (5, 5, 1, 2), (5, 5, 2, 2)):
    L = lfa._cell(p, q, s)
    n = nk * L
    t0 = time.time()
    got = pkg.lfa_torus(p, q, n, s, h_factor=2, iters=300, seed=5, dim=3)
    print(f"{p:2d} {q:2d} {s:2d} {nk:3d} {n:4d} {got:9.5f}  ({time.time() - t0:.1f} s, {n ** 3} DOF)", flush=True)
print()
print("at scale (the torus alone, no oracle): n = 32 L")
for p in (3, 5, 8):
    s = S[p]
    n = 32 * (s + p)
    t0 = time.time()
    got = pkg.lfa_torus(p, 1, n, s, h_factor=1, iters=300, seed=3)
    print(f"{p:2d} 1 {s:2d}  32 {n:4d} {got:9.5f}  ({time.time() - t0:.1f} s, {n * n} DOF)", flush=True)
