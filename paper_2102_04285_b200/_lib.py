"""ctypes binding of the C ABI in ``include/xstrace_b200.h``.

The shared library is built in-tree (``paper_2102_04285_b200/libxstrace_b200.so``,
see ``csrc/build.sh``).  There is no fallback: if the library or a CUDA
device is missing, every analysis entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XS_LIB_PATH") or os.path.join(HERE, "libxstrace_b200.so")  # (override: A/B experiments)

XS_OK = 0
XS_INVALID_TRACE = 1
XS_UNCALIBRATED = 2
XS_CUDA_ERROR = 3
XS_BAD_ARGUMENT = 4
XS_UNSUPPORTED = 5
XS_NO_MEMORY = 6


class XsEvents(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("start", C.c_void_p), ("dur", C.c_void_p), ("pid", C.c_void_p), ("tid", C.c_void_p),
        ("cat", C.c_void_p), ("name", C.c_void_p), ("corr", C.c_void_p), ("has_corr", C.c_void_p),
        ("n_pids", C.c_int32), ("n_groups", C.c_int32), ("n_names", C.c_int32), ("reserved", C.c_int32),
        ("group_pid", C.c_void_p), ("pid_has_meta", C.c_void_p),
    ]


class XsPacked(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("row0", C.c_int64),
        ("start", C.c_void_p), ("start_base", C.c_void_p), ("dur", C.c_void_p), ("pid", C.c_void_p),
        ("tid", C.c_void_p), ("name", C.c_void_p), ("corr", C.c_void_p), ("catf", C.c_void_p),
        ("start_w", C.c_int32), ("dur_w", C.c_int32), ("pid_w", C.c_int32), ("tid_w", C.c_int32),
        ("name_w", C.c_int32), ("corr_w", C.c_int32),
        ("n_exc", C.c_int64), ("exc_row", C.c_void_p), ("exc_val", C.c_void_p), ("exc_col", C.c_void_p),
    ]


class XsPackLayout(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("n_exc", C.c_int64), ("total", C.c_int64),
        ("start_w", C.c_int32), ("dur_w", C.c_int32), ("corr_w", C.c_int32), ("pid_w", C.c_int32),
        ("tid_w", C.c_int32), ("name_w", C.c_int32), ("n_threads", C.c_int32), ("reserved", C.c_int32),
        ("offset", C.c_int64 * 13), ("nbytes", C.c_int64 * 13), ("thread_exc", C.c_int64 * 64),
    ]


class XsSynthSpec(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64), ("seed", C.c_uint64), ("n_pids", C.c_int32), ("outer_op", C.c_int32),
        ("second_tid_ops", C.c_int32), ("first_pid", C.c_int32), ("ann_start", C.c_int64), ("ann_end", C.c_int64),
        ("transition", C.c_int64), ("interception", C.c_int64), ("launch", C.c_int64), ("memcpy", C.c_int64),
        ("names", C.c_void_p),
    ]


class XsProfile(C.Structure):
    _fields_ = [
        ("words", C.c_int32), ("reserved", C.c_int32), ("L", C.c_void_p), ("whole", C.c_int64 * 4),
        ("frac", C.c_void_p), ("internal", C.c_void_p), ("has_internal", C.c_void_p),
        ("residue_in", C.c_void_p), ("span_end_in", C.c_void_p),
    ]


class XsOverlapInfo(C.Structure):
    _fields_ = [("n_cells", C.c_int64), ("n_nodes", C.c_int32), ("n_pids", C.c_int32)]


class XsCorrectInfo(C.Structure):
    _fields_ = [("original_total", C.c_int64), ("corrected_total", C.c_int64),
                ("n_sites", C.c_int64), ("n_slabs", C.c_int64)]


# every exported symbol with its (restype, argtypes); tests check the .so
# exports exactly what the header declares
P = C.c_void_p
SIGNATURES = {
    "xs_status_str": (C.c_char_p, [C.c_int]),
    "xs_last_error": (C.c_char_p, [P]),
    "xs_version": (C.c_int, []),
    "xs_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "xs_ctx_destroy": (None, [P]),
    "xs_ctx_workspace_bytes": (C.c_int64, [P]),
    "xs_validate": (C.c_int, [P, C.POINTER(XsEvents), C.POINTER(C.c_int64), P]),
    "xs_overlap": (C.c_int, [P, C.POINTER(XsEvents), C.c_int, P]),
    "xs_overlap_info": (C.c_int, [P, C.POINTER(XsOverlapInfo)]),
    "xs_overlap_fetch": (C.c_int, [P, P, P, P, P, P, P, P, P, P, P, P]),
    "xs_correct": (C.c_int, [P, C.POINTER(XsEvents), C.POINTER(XsProfile), P, P, C.POINTER(C.c_int64), P]),
    "xs_correct_report": (C.c_int, [P, C.POINTER(XsCorrectInfo), P, P, P]),
    "xs_remap": (C.c_int, [P, C.c_int64, P, P, P, P]),
    "xs_analyze": (C.c_int, [P, C.POINTER(XsEvents), C.POINTER(XsProfile), C.c_int, P, P,
                             C.POINTER(C.c_int64), P]),
    "xs_analyze_to_host": (C.c_int, [P, C.POINTER(XsEvents), C.POINTER(XsProfile), C.c_int, P, P, P, P,
                                     C.POINTER(C.c_int64), P]),
    "xs_analyze_to_host_async": (C.c_int, [P, C.POINTER(XsEvents), C.POINTER(XsProfile), C.c_int, P, P, P, P,
                                           C.POINTER(C.c_int64), P]),
    "xs_host_copy_wait": (C.c_int, [P]),
    "xs_transition_sites": (C.c_int, [P, C.POINTER(XsEvents), C.c_int, C.POINTER(C.c_int64), P]),
    "xs_transition_fetch": (C.c_int, [P, P, P, P]),
    "xs_union": (C.c_int, [P, C.POINTER(XsEvents), C.c_int, C.c_int, P, C.POINTER(C.c_int64),
                           C.POINTER(C.c_int64), P]),
    "xs_utilization": (C.c_int, [P, C.POINTER(XsEvents), C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64), C.POINTER(C.c_int64), P]),
    "xs_union_intervals_fetch": (C.c_int, [P, P, P, P]),
    "xs_chunk_info": (C.c_int, [P, C.c_int64, C.c_char_p, P, P, P, C.c_char_p, C.c_int]),
    "xs_chunk_decode": (C.c_int, [P, C.c_int64, C.c_char_p, P, P, P, P, P, P, P, P, P, P, C.c_char_p, C.c_int]),
    "xs_unpack": (C.c_int, [P, P, P, P, P, P, P, P, P, P, P]),
    "xs_pack_plan": (C.c_int, [C.POINTER(XsEvents), C.c_int, C.POINTER(XsPackLayout)]),
    "xs_pack_fill": (C.c_int, [C.POINTER(XsEvents), C.POINTER(XsPackLayout), P, C.c_int64]),
    "xs_synth_plan": (C.c_int, [P, C.POINTER(XsSynthSpec), C.POINTER(C.c_int64), P]),
    "xs_synth_generate": (C.c_int, [P, C.POINTER(XsSynthSpec), P, P, P, P, P, P, P, P, P, P, P, P]),
    "xs_launch_count": (C.c_int64, [P]),
    "xs_profile_enable": (C.c_int, [P, C.c_int]),
    "xs_profile_read": (C.c_int, [P, P, P, C.c_int]),
    "xs_profile_stage_name": (C.c_char_p, [C.c_int]),
}

_lib = None


def load():
    """Load the CUDA library or fail loudly (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"xstrace-b200 CUDA library not built: {LIB_PATH} is missing "
                "(run paper_2102_04285_b200/csrc/build.sh or __graft_entry__.build())"
            )
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
