"""Block-LFA two-grid factors of the multicolour two-level method (oracle/lfa.py; exact second level at
the same h, Table 1's setting) for the paper's block choices and the bench configs' (p, q, d):
python tools/lfa_table.py > profiles/lfa_r01.txt  (CPU only; calls nothing but oracle/)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.lfa import rho_2g  # noqa: E402

cases = [(2, 1, 3, 2, 8), (3, 1, 3, 2, 8), (4, 1, 3, 2, 8), (5, 1, 5, 2, 8), (6, 1, 5, 2, 6), (7, 1, 7, 2, 4),
         (8, 1, 7, 2, 4), (8, 2, 7, 2, 4), (5, 2, 5, 2, 6), (2, 1, 3, 3, 4), (3, 1, 3, 3, 4)]
print("p q s d  nk^d  rho_2g (multicolour block LFA, exact q-level solve at h)")
for p, q, s, d, nk in cases:
    t = time.time()
    r = rho_2g(p, q, s, d, nk=nk)
    print(f"{p} {q} {s} {d}  {nk}^{d}  {r:.4f}   ({time.time() - t:.1f} s)", flush=True)
