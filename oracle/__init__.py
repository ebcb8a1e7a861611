"""FP64 CPU oracle for the box-spline parallel-beam CT hot path (arXiv 2005.13471).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import anything from this package.  The
product (paper_2005_13471_b200/) never imports it, and it never imports the
product: the two share no code (only the seeded input generators in synth/).

Plain, slow, obviously-correct NumPy in float64, written from PAPER.md (cited as
P:<line>).  Each function follows the paper's definition or algorithm in the
paper's order; library primitives used as steps: numpy/scipy FFT (normal apply at
large N, pinned against the direct Toeplitz sum), numpy.linalg (dense solves in
tests).  Readings where the paper is silent/ambiguous are SURVEY.md R1-R20 and are
listed in DESIGN.md.

Modules
  boxspline   M_W(x), Eq.(1)-(2)                      pinned: tests/test_oracle_boxspline.py
  geometry    lattice, detector grid, projected widths pinned via gram/forward pins
  gram        Gram taps P:96-131; brute-force H^T H    pinned: tests/test_oracle_gram.py
  normal      Toeplitz apply (direct, FFT) P:131       pinned: tests/test_oracle_normal.py
  backproject correction filter Eq.(5), H^T g^         pinned: tests/test_oracle_backproject.py
  forward     H c, Eq.(3)-(4); geometric footprints;   pinned: tests/test_oracle_forward.py
              plain adjoint H^T (dot-product test)
  solvers     CG / steepest descent / Landweber        pinned: tests/test_oracle_solvers.py
  sirt        SIRT on H / H^T (NEXT-1)                 pinned: tests/test_oracle_sirt.py
Parity unpinned: none of the functions above (every one has an independent pin);
the FP32 CG iterate itself is chaotic -- see DESIGN.md.
"""
