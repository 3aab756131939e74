"""CPU oracle for the BT/BTA SI+SQ hot path -- TEST INFRASTRUCTURE ONLY.

This package is a NumPy/SciPy restatement of the reference algorithm
(`btasel`, /root/reference/pkg/src/btasel), written independently and citing
the reference file:line each function follows.  It is the *checker*:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
  leg (``cpu_baseline`` / ``--impl reference``) may import it;
* the product package ``paper_2601_04904_b200`` never imports it and has no
  CPU fallback -- it fails loudly when its CUDA library is missing.

Parity pinning: the restatement is checked against golden vectors produced
by running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) and against the
reference's own known-answer tests (tests/test_oracle_golden.py).
"""

from .seq import (  # noqa: F401
    OracleSingular,
    Blocks,
    generate_dd_bta,
    hermitianize,
    to_dense,
    mask_to_pattern,
    dense_selected,
    forward,
    backward,
    solve_selected,
    op_counts,
)
from .dist import plan_partitions, dist_solve  # noqa: F401
