"""CPU ORACLE for the BB-preconditioned Newton-system solve (arXiv 2209.00315).

*** TEST INFRASTRUCTURE ONLY. ***  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import anything under
`oracle/`.  The product path (`paper_2209_00315_b200`) never imports it and
shares no code, headers, helpers or constants with it; it fails loudly if its
CUDA library is missing.

A plain, slow, obviously-correct fp64 implementation written from PAPER.md,
in the paper's order and notation, with scipy.sparse / numpy as the library
primitives (sparse products, dense solves).  Citation keys: P:n = PAPER.md
line n; S:n = SPEC.md line n; A-numbers are the readings of SURVEY.md §8(c)
(restated in DESIGN.md §2).

  mesh.py    D1-D2  two-level TPFA geometry
  ops.py     D2-D12 operators, residuals (2.5)-(2.7), Jacobian blocks (3.1),
                    projected system (4.17), BB operators Ã, B̃, T (4.22)-(4.26)
  amg.py     I3     pairwise-aggregation AMG (build decision, PARITY UNPINNED by the paper)
  krylov.py  I1,I4,I5  FGMRES, per-slice PCG, GMRES(10)
  bb.py      I2, a6 BB preconditioner apply (4.18)-(4.20)+(4.26), recovery (4.15)
  simple.py  f1     SIMPLE preconditioner on (eq:saddle-point), NEXT row
  hss.py     f2     HSS preconditioner (eq:prec-hss), NEXT row
  ipm.py     a7     interior-point loop
  direct.py         dense direct solve of (3.1) for tiny instances (pin)

Pins (tests/test_oracle_*.py) tie every function to something other than
itself: counting identities, the adjoint identity div = -grad^T diag(|w||e|),
Remark 2.2 mass conservation, a central finite-difference Jacobian, the kernel
of J (Remark 3.1), projector identities, exact-inner-solve BB -> 2 FGMRES
iterations, dense direct solves, closed-form kinetic energy of a translation,
and the IPM central-path gap.  The AMG internals (I3) have no paper pin:
"parity unpinned".
"""
