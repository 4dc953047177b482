"""B200-native ABFT-protected blocked factorizations (Cholesky / LU / QR).

A drop-in for the hot path of the reference `slackwise` package
(SURVEY.md §8): the same Python names and semantics, backed by hand-written
sm_100a kernels in ``libabft_b200.so`` through a C-ABI
(``include/abft_b200.h``). There is no CPU fallback.
"""
from .abft import (CHECK_TOLERANCE_FACTOR, INDEX_SNAP_TOLERANCE, ChecksumScheme,  # noqa: F401
                   CorrectionReport, ErrorKind, InjectedFault, RegionChecksums,
                   checksum_flops, encode, inject_faults, maintain_gemm,
                   sample_fault_plan, verify_correct)
from .linalg import (BlockLayout, DecompositionKind, Factorization,  # noqa: F401
                     InvalidDimensionError, NumericBreakdownError, TaskKind,
                     algorithmic_flops, compute_flops, generate_test_matrix, residual,
                     touched_elements)
from .simulator import (CORRECTNESS_RESIDUAL, run_numeric_iteration,  # noqa: F401
                        run_protected)
from .install import install, uninstall  # noqa: F401
from .single import SFactorization  # noqa: F401  (fp32 s* variants on tcgen05)
from . import governor  # noqa: F401  (run modes / adaptive ABFT / slack reclamation)

__version__ = "0.1.0"
