"""Block-LFA factors of the multicolour two-level method (oracle/lfa.py): two-grid with the
exact second level at the same h (rho_2g, Table 1's setting), three-grid with one q-level two-grid cycle
(rho_3g, Table 2's setting) and the aggressive two-grid on H = 2h (rho_2g^ag, Table 3's setting), for the
paper's block choices and the bench configs' (p, q, d):
python tools/lfa_table.py > profiles/lfa_r02.txt  (CPU only; calls nothing but oracle/)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.lfa import rho_2g, rho_2g_ag, rho_3g  # noqa: E402

cases = [(2, 1, 3, 2, 4), (3, 1, 3, 2, 4), (4, 1, 3, 2, 4), (5, 1, 5, 2, 4), (6, 1, 5, 2, 4), (7, 1, 7, 2, 2),
         (8, 1, 7, 2, 2), (8, 2, 7, 2, 2), (5, 2, 5, 2, 4)]
print("p q s d  nk^d  rho_2g   rho_3g   rho_2g^ag  (multicolour block LFA)")
for p, q, s, d, nk in cases:
    t = time.time()
    r2, r3, ra = rho_2g(p, q, s, d, nk=nk), rho_3g(p, q, s, d, nk=nk), rho_2g_ag(p, q, s, d, nk=nk)
    print(f"{p} {q} {s} {d}  {nk}^{d}  {r2:.4f}   {r3:.4f}   {ra:.4f}     ({time.time() - t:.1f} s)", flush=True)
