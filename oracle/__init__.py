"""CPU ORACLE for the monolithic multigrid hot path of arXiv 2107.04060.

*** TEST INFRASTRUCTURE ONLY ***  Only ``tests/`` (incl. the golden-record scripts in
``tests/scripts/``), ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or
run anything in this package.  The product path (``paper_2107_04060_b200``)
never imports it, and this package never imports the product path: the two
share no code, tables or constants.  The only shared module is ``mg_inputs``,
which draws seeded inputs and holds none of the method's arithmetic.

The oracle is plain, slow and literal: global sparse assembly of the blocks of
PAPER.md eq. (block_form_rq), explicit dense per-patch solves for Vanka, the
paper's two-stage inexact Braess-Sarazin update, the column-wise
divergence-preserving interpolation of PAPER.md §3.1, and a recursive V-cycle
(PAPER.md eq. (TG-Operator-Biot)).  Everything is IEEE fp64.

Modules
  mesh      structured triangulation, DoF slots, incidence
  fem       element integrals and the assembled operator A^RQ
  transfer  P_u (divergence preserving), P_w, P_p, R = P^T
  relax     additive Vanka and inexact BSR
  cycle     hierarchy, coarsest solve, V-cycle, stationary solve, rho_N
  manufactured  steady manufactured problem and FE error norms
  lfa       two-grid local Fourier analysis from the assembled stencils

Pins: every function here is checked by ``tests/test_oracle_*.py`` against
something the paper or mathematics fixes (Appendix A stencils, Appendix B
transfer sums, exact Galerkin identities, brute-force dense two-grid
operators, the printed two-grid convergence factors of tab:vanka22 and
tab:bsr_vanka11, their printed LFA predictions rho_LFA (all 72 cells
within 1e-3, which pins A_h, A_H, P, Vanka and BSR on the infinite grid), FE
convergence rates).  Functions without such a pin are
marked "parity unpinned" in their docstring and in DESIGN.md.
"""
