"""CPU-only checks of the boundary: the sm_100a library loads, exports every
symbol include/abft_b200.h declares, the ctypes table matches the header,
and the host-side logic (RNG draws, regions, flop model) equals the
reference's (goldens). No compute calls: there is no GPU here."""
import re

import numpy as np
import pytest

import paper_2301_03166_b200 as P
from paper_2301_03166_b200 import _lib
from conftest import ROOT, golden

HEADER = ROOT / "include" / "abft_b200.h"


def header_symbols():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"ABFT_API\s+[\w\s\*]+?\b(abft_\w+)\s*\(", txt)))


def test_library_builds_and_exports_header():
    from paper_2301_03166_b200.build import build_library
    path = build_library()
    import ctypes
    lib = ctypes.CDLL(str(path))
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s


def test_ctypes_table_matches_header():
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == header_symbols()


def test_library_typed_load_and_version():
    lib = _lib.load()
    assert lib.abft_version() >= 100


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(_lib.LibraryUnavailable):
        _lib.load(tmp_path / "nope.so")


def test_struct_layouts_match_header(tmp_path):
    """ctypes structs == the C compiler's layout of the header structs."""
    import ctypes
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no C compiler")
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "abft_b200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(abft_fault),'
                   ' sizeof(abft_location), sizeof(abft_report), offsetof(abft_fault, magnitude),'
                   ' offsetof(abft_location, seq), offsetof(abft_report, n_locations));return 0;}')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", f"-I{HEADER.parent}", str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(_lib.Fault), ctypes.sizeof(_lib.Location),
                   ctypes.sizeof(_lib.Report), _lib.Fault.magnitude.offset,
                   _lib.Location.seq.offset, _lib.Report.n_locations.offset]


def test_sample_fault_plan_matches_reference():
    g = golden("plans.json")
    rng = np.random.default_rng(11)
    E = P.ErrorKind
    for want in g["small"]:
        plan = P.sample_fault_plan(rng, {E.D0: 1, E.D1: 1, E.D2: 1}, r0=8, c0=8, rows=24, cols=24,
                                   b=8, scale=1.0, iteration=0)
        assert [[f.kind.value, f.row, f.col, f.magnitude, f.extent, f.orientation]
                for f in plan] == want
    rng = np.random.default_rng(5)
    for scale, want in zip((0.3, 3.7, 1234.5), g["big"]):
        plan = P.sample_fault_plan(rng, {E.D0: 3, E.D1: 2, E.D2: 2}, r0=256, c0=512, rows=7936,
                                   cols=7680, b=256, scale=scale, iteration=1)
        assert [[f.kind.value, f.row, f.col, f.magnitude, f.extent, f.orientation]
                for f in plan] == want


def test_generate_test_matrix_bit_exact():
    import hashlib
    for case in golden("inputs.json"):
        a = P.generate_test_matrix(case["kind"], case["n"], case["seed"])
        assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == case["sha256"]
    with pytest.raises(P.InvalidDimensionError):
        P.generate_test_matrix("lu", 0, 1)


def test_block_layout_and_regions():
    lay = P.BlockLayout(100, 32)
    assert lay.n_blocks == 4 and lay.block_slice(3) == slice(96, 100)
    with pytest.raises(P.InvalidDimensionError):
        P.BlockLayout(10, 11)
    from paper_2301_03166_b200.simulator import _tmu_region
    import oracle as O
    for kind in ("cholesky", "lu", "qr"):
        for n, b in ((100, 32), (256, 256), (2048, 256)):
            for k in range(-(-n // b)):
                assert _tmu_region(kind, n, b, k) == O.region_of(kind, n, b, k)


@pytest.mark.parametrize("kind", ["cholesky", "lu", "qr"])
def test_flop_model_closed_forms(kind):
    n, b = 512, 64
    total = sum(P.compute_flops(kind, t, n, b, k) for k in range(n // b) for t in ("pd", "pu", "tmu"))
    assert total == pytest.approx(P.algorithmic_flops(kind, n), rel=3.0 * b / n)


def test_checksum_cost_model():
    assert P.checksum_flops("none", "lu", "tmu", 256, 32, 0) == 0.0
    f = P.compute_flops("lu", "tmu", 256, 32, 0)
    assert P.checksum_flops("single", "lu", "tmu", 256, 32, 0) == 2.0 * f / 32
    assert P.checksum_flops("full", "lu", "tmu", 256, 32, 0) == 4.0 * f / 32


def test_encode_rejects_none_scheme():
    with pytest.raises(ValueError):
        P.RegionChecksums(0, 0, (4, 4), 2, "none")


def test_install_patches_reference_when_present():
    try:
        import sys
        sys.path.insert(0, "/root/reference/pkg/src")
        import slackwise  # noqa: F401
    except ImportError:
        pytest.skip("reference package not present on this machine")
    import slackwise
    import slackwise.simulator as sim
    orig = sim.run_numeric_iteration
    assert P.install()
    try:
        assert sim.run_numeric_iteration is P.run_numeric_iteration
        assert sim.Factorization is P.Factorization
        assert slackwise.residual is P.residual
        assert P.linalg.ERRORS["breakdown"] is slackwise.NumericBreakdownError
    finally:
        P.uninstall()
    assert sim.run_numeric_iteration is orig
