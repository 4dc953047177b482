"""ctypes binding of libabft_b200.so (include/abft_b200.h).

There is no CPU fallback: if the sm_100a library is missing or cannot be
loaded, every compute entry point raises. The library is built in-tree by
``paper_2301_03166_b200.build`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libabft_b200.so"

# error codes (abft_b200.h)
OK = 0
E_INVALID = -1
E_DIM = -2
E_BREAKDOWN = -3
E_RANGE = -4
E_INCOMPLETE = -5
E_OVERFLOW = -6

KIND_CODE = {"cholesky": 0, "lu": 1, "qr": 2}
SCHEME_CODE = {"none": 0, "single": 1, "full": 2}
ERROR_NAME = ("0d", "1d", "2d")
TASK_CODE = {"pd": 0, "pu": 1, "tmu": 2}


class Fault(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("orientation", ctypes.c_int32),
                ("row", ctypes.c_int64), ("col", ctypes.c_int64),
                ("extent", ctypes.c_int32), ("absolute", ctypes.c_int32),
                ("u", ctypes.c_double), ("negate", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("magnitude", ctypes.c_double)]


class Location(ctypes.Structure):
    _fields_ = [("row", ctypes.c_int64), ("col", ctypes.c_int64), ("kind", ctypes.c_int32),
                ("flag", ctypes.c_int32), ("detected_kind", ctypes.c_int32),
                ("corrected", ctypes.c_int32), ("uncorrectable", ctypes.c_int32),
                ("block_row", ctypes.c_int32), ("block_col", ctypes.c_int32),
                ("seq", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("detected", ctypes.c_int64 * 3), ("corrected", ctypes.c_int64 * 3),
                ("uncorrectable", ctypes.c_int32), ("n_locations", ctypes.c_int32)]


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_F = ctypes.POINTER(ctypes.c_float)
_I64 = ctypes.c_int64
_I = ctypes.c_int

# (name, restype, argtypes) — every symbol declared in include/abft_b200.h
SIGNATURES = [
    ("abft_version", _I, []),
    ("abft_last_error", ctypes.c_char_p, []),
    ("abft_device_count", _I, [ctypes.POINTER(_I)]),
    ("abft_launch_count", ctypes.c_longlong, []),
    ("abft_noise_stats", _I, [_I]),
    ("abft_noise_read", _I, [_D, _I]),
    ("abft_dev_dgemm", _I, [_P, ctypes.c_char, ctypes.c_char, _I64, _I64, _I64, ctypes.c_double,
                            _P, _I64, _P, _I64, ctypes.c_double, _P, _I64, _P, _I64]),
    ("abft_dev_sgemm", _I, [_P, ctypes.c_char, ctypes.c_char, _I64, _I64, _I64, ctypes.c_float,
                            _P, _I64, _P, _I64, ctypes.c_float, _P, _I64, _P, _I64]),
    ("abft_dev_sgemm_splitk", _I, [_P, ctypes.c_char, ctypes.c_char, _I64, _I64, _I64,
                                   ctypes.c_float, _P, _I64, _P, _I64, ctypes.c_float, _P, _I64,
                                   _P, _I64, _I]),
    ("abft_dev_diag_factor", _I, [_P, _I, _I, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _P]),
    ("abft_dev_sdiag_factor", _I, [_P, _I, _I, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _P]),
    ("abft_create", _I, [ctypes.POINTER(_P), _I, _I64, _I64, _I]),
    ("abft_destroy", _I, [_P]),
    ("abft_set_matrix", _I, [_P, _D, _I64]),
    ("abft_set_matrix_streamed", _I, [_P, _D, _I64]),
    ("abft_keep_input", _I, [_P, _I]),
    ("abft_reset", _I, [_P]),
    ("abft_stream", _P, [_P]),
    ("abft_make_spd", _I, [_P]),
    ("abft_get_matrix", _I, [_P, _D, _I64]),
    ("abft_k_done", _I64, [_P]),
    ("abft_set_k_done", _I, [_P, _I64]),
    ("abft_task", _I, [_P, _I64, _I]),
    ("abft_iteration", _I, [_P, _I64, _I, ctypes.POINTER(Fault), _I, _I, ctypes.POINTER(Report),
                            ctypes.POINTER(Location), _I]),
    ("abft_factorize", _I, [_P, _I, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(Fault),
                            ctypes.POINTER(ctypes.c_int64), _I, _I, ctypes.POINTER(Report),
                            ctypes.POINTER(Location), _I, ctypes.POINTER(_I)]),
    ("abft_stream_out", _I, [_P, _D, _I64]),
    ("abft_qr_panels", _I, [_P]),
    ("abft_set_qr_panels", _I, [_P, _I]),
    ("abft_get_qr_panel", _I, [_P, _I64, _D, _I64, _D, _I64]),
    ("abft_profile", _I, [_P, _I]),
    ("abft_profile_read", _I, [_P, _D]),
    ("abft_profile_read_iters", _I, [_P, _D, _I64]),
    ("abft_set_side_sms", _I, [_P, ctypes.POINTER(ctypes.c_int32), _I64]),
    ("abft_set_input_chunks", _I, [_P, _I, _I64, _I]),
    ("abft_s_set_input_chunks", _I, [_P, _I, _I64, _I]),
    ("abft_set_pivoting", _I, [_P, _I]),
    ("abft_get_pivots", _I, [_P, ctypes.POINTER(ctypes.c_int32)]),
    ("abft_probe_dmma_peak", _I, [_I, _D]),
    ("abft_snapshot", _I, [_P, _I]),
    ("abft_restore", _I, [_P, _I]),
    ("abft_residual", _I, [_P, _D, _I64, _D]),
    ("abft_reconstruct", _I, [_P, _D, _I64]),
    ("abft_breakdown_column", _I64, [_P]),
    ("abft_debug_array", _I, [_P, _I, _D, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("abft_last_elapsed_ms", _I, [_P, _D]),
    ("abft_dist_create", _I, [ctypes.POINTER(_P), _I, _I64, _I64, _I, _I, _I]),
    ("abft_dist_destroy", _I, [_P]),
    ("abft_dist_local_cols", _I64, [_P]),
    ("abft_dist_stream", _P, [_P]),
    ("abft_dist_xbuf_elems", _I64, [_P, _I64]),
    ("abft_dist_set_matrix", _I, [_P, _D, _I64]),
    ("abft_dist_get_matrix", _I, [_P, _D, _I64]),
    ("abft_dist_set_local", _I, [_P, _D, _I64]),
    ("abft_dist_keep_input", _I, [_P, _I]),
    ("abft_dist_reset", _I, [_P]),
    ("abft_dist_begin", _I, [_P, _I64, _I, _P]),
    ("abft_dist_exchange", _I, [_P, _I64, ctypes.POINTER(_I)]),
    ("abft_dist_update", _I, [_P, _I64, _I, _P, _I, _P]),
    ("abft_dist_finish", _I, [_P, _I64, _I, ctypes.POINTER(Fault), _I, _I, _P]),
    ("abft_dist_events", _I, [_P, ctypes.POINTER(Location), ctypes.POINTER(_I64), _I,
                              ctypes.POINTER(_I)]),
    ("abft_dist_k_done", _I64, [_P]),
    ("abft_dist_get_qr_panel", _I, [_P, _I64, _D, _I64, _D, _I64]),
    ("abft_dist_elapsed_ms", _I, [_P, _D]),
    ("abft_dist_lookahead", _I, [_P, _I64, _P]),
    ("abft_dist_comm_stream", _P, [_P]),
    ("abft_dist_comm_done", _I, [_P]),
    ("abft_set_qr_panel", _I, [_P, _I64, _D, _I64, _D, _I64]),
    ("abft_s_create", _I, [ctypes.POINTER(_P), _I, _I64, _I64, _I]),
    ("abft_s_destroy", _I, [_P]),
    ("abft_s_stream", _P, [_P]),
    ("abft_s_k_done", _I64, [_P]),
    ("abft_s_keep_input", _I, [_P, _I]),
    ("abft_s_set_matrix", _I, [_P, _F, _I64]),
    ("abft_s_set_matrix_streamed", _I, [_P, _F, _I64]),
    ("abft_s_reset", _I, [_P]),
    ("abft_s_make_spd", _I, [_P]),
    ("abft_s_get_matrix", _I, [_P, _F, _I64]),
    ("abft_s_iteration", _I, [_P, _I64, _I, ctypes.POINTER(Fault), _I, _I, ctypes.POINTER(Report),
                              ctypes.POINTER(Location), _I]),
    ("abft_s_factorize", _I, [_P, _I, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(Fault),
                              ctypes.POINTER(ctypes.c_int64), _I, _I, ctypes.POINTER(Report),
                              ctypes.POINTER(Location), _I, ctypes.POINTER(_I)]),
    ("abft_s_last_elapsed_ms", _I, [_P, _D]),
    ("abft_s_stream_out", _I, [_P, _F, _I64]),
    ("abft_s_snapshot", _I, [_P]),
    ("abft_s_restore", _I, [_P]),
    ("abft_s_profile", _I, [_P, _I]),
    ("abft_s_profile_read", _I, [_P, _D]),
    ("abft_s_residual", _I, [_P, _F, _I64, _D]),
    ("abft_s_breakdown_column", _I64, [_P]),
    ("abft_region_encode", _I, [_D, _I64, _I64, _I64, _I64, _I, _D, _D, _D, _D]),
    ("abft_region_maintain", _I, [_I64, _I64, _I64, _I64, _I, _D, _I64, _D, _I64, _D, _D, _D,
                                  _D]),
    ("abft_region_verify", _I, [_D, _I64, _I64, _I64, _I64, _I, _I, _I64, _I64, _D, _D, _D,
                                ctypes.POINTER(Report), ctypes.POINTER(Location), _I]),
    ("abft_inject", _I, [_D, _I64, _I64, _I64, ctypes.POINTER(Fault), _I, ctypes.c_double]),
]

_lock = threading.Lock()
_lib = None


class LibraryUnavailable(RuntimeError):
    pass


def load(path: str | os.PathLike | None = None):
    """Load (once) and type the shared library. Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # ABFT_LIB: an alternative build of the same library (A/B measurements)
        p = Path(path) if path else Path(os.environ.get("ABFT_LIB", str(LIB_PATH)))
        if not p.exists():
            raise LibraryUnavailable(
                f"{p} not found: build it with `python -m paper_2301_03166_b200.build` "
                "(the B200 path has no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    msg = load().abft_last_error()
    return msg.decode(errors="replace") if msg else ""


def dptr(a) -> "ctypes._Pointer":
    return a.ctypes.data_as(_D)


def fptr(a) -> "ctypes._Pointer":
    return a.ctypes.data_as(_F)
