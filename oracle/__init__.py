"""fp64 CPU oracle for the facet-consensus deblurring hot path.

THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import, call, link or
execute anything under oracle/.  The product path (paper_1705_06603_b200/)
never imports it and shares no code with it.

Contents (each function cites the PAPER.md passage it follows):
  oracle.c / operators.py  H and H^T as literal double sums
  geometry.py              facet index sets and omega^F
  tv.py                    D, phi, psi (smoothed TV / Huber)
  solver.py                Algorithm 1 with Lemma 1
  vmlmb.py                 VMLM-B Local-Solver (reading V1-V6) PAPER.md:287, :290

Pins (tests/test_oracle_*.py, -m "not gpu") tie every function to something
other than itself; see DESIGN.md §4 for the table.  No function here is
"parity unpinned".  The paper prints no values for the BASELINE configs (their
inputs are synthetic), so the absolute iterate / objective values there rest on
the structural pins (single facet = centralized projected gradient, fixed
point = consensus-reduced minimiser, exact-arithmetic trace).
"""
from . import geometry, tv  # noqa: F401
from .operators import Operator  # noqa: F401
from .solver import Deblur, Params, default_tau, from_problem, consensus, dr_iteration  # noqa: F401
