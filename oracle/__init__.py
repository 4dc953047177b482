"""CPU oracle for the ABFT-protected blocked factorization hot path.

TEST INFRASTRUCTURE ONLY. Nothing in the product (``paper_2301_03166_b200``)
imports, links or executes this package; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs use it, and only as the checker or as the timed
CPU reference arm.

It restates, in numpy, the reference algorithm of the `slackwise` package
(/root/reference/pkg/src/slackwise/, pure Python) for the hot path named in
SURVEY.md §8: the blocked Cholesky / LU / QR numeric engine
(linalg.py:159-368), the block-checksum ABFT primitives (abft.py:87-333) and
the protected iteration (simulator.py:86-167). Each function cites the
reference lines it follows.

Parity pinning: the oracle is checked against golden vectors produced by
running the reference itself in this container
(``tests/golden/make_golden.py`` → ``tests/golden/*.json``); see
``tests/test_oracle_golden.py``.
"""

from .abft_oracle import (  # noqa: F401
    CHECK_TOLERANCE_FACTOR, INDEX_SNAP_TOLERANCE, ALL_KINDS, ERROR_KINDS,
    OracleFactorization, OracleReport, Checksums, block_sums, draw_fault_plan,
    encode, generate_test_matrix, inject, magnitude, maintain, protected_iteration,
    region_of, residual, verify, algorithmic_flops,
)
