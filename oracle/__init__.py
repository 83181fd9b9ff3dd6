"""ORACLE — plain, slow, CPU-only reference for the two-level IGA iteration.

THIS PACKAGE IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call or execute anything in here.  The
product path (``paper_2009_01499_b200`` + ``libiga2l.so``) never touches it
and shares no code, tables or constants with it.

It is written straight from the paper (arXiv 2009.01499, /root/reference/PAPER.md,
cited as ``P:<line>``) in fp64 with NumPy/SciPy; every function cites the
passage it follows.  Where the paper is silent the reading taken is the one in
SURVEY.md §8(c) (cited as ``A<n>``) and listed in DESIGN.md.

Modules
-------
bspline    knot vector, Cox–de Boor recursion, derivatives, Gauss rules
assembly   1D K/M, cross mass, d-dim sparse Galerkin stiffness, load
transfer   lumped L2-projection degree transfer, knot-insertion mesh transfer
schwarz    overlapping multiplicative Schwarz: lex and multicolour orders
multigrid  multicolour Gauss–Seidel V(1,1) on the q-level
twolevel   Algorithm 1, solve loop, asymptotic rate, dense error operator
lfa        block local Fourier analysis of the multicolour two-grid         (reading A28)

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``.  Table 4 iteration
counts are "parity unpinned": no ordering we can
build reproduces them, so they are context only.
"""
