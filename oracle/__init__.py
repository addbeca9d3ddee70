"""CPU oracle for the polygrain fit hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain NumPy fp64, the reference algorithm of
``polygrain.objective.evaluate_objective`` / ``hard_assign`` (the hot path
named by BASELINE.json ``north_star``) together with the pieces it consumes
(grid coordinates, graded-lex Legendre/monomial design features, tie-tolerant
arg-min).  It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may
import it.  The product package ``paper_2605_20816_b200`` never imports it and
fails loudly when its CUDA library is missing.

Parity pinning: every function here is checked against golden vectors that
were produced by running the *reference itself* (``/root/reference/pkg``,
imported read-only in the build container) — see
``tests/golden/make_golden.py`` and ``tests/test_oracle_golden.py``.  The
3-D basis/grid and the lambda term are extensions the reference does not have
(SURVEY.md Appendix B); they reduce to the reference at their neutral setting
and are pinned by the 2-D-embedding cross-check instead.
"""

from .polygrain_oracle import *  # noqa: F401,F403
