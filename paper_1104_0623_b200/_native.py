"""ctypes binding of the C ABI declared in include/find_b200.h.

This is the whole host<->native boundary: plain pointers, sizes and a CUDA
stream handle; no torch types.  The library is built in-tree by
``paper_1104_0623_b200.build`` and there is no fallback: if it is missing the
import fails loudly.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import NativeLibraryError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libfind_b200.so"

FIND_OK, FIND_EINVAL, FIND_ESINGULAR, FIND_ECUDA, FIND_ENOMEM = 0, 1, 2, 3, 4
LEDGER_KEYS = 12

# every symbol include/find_b200.h declares
EXPORTED = (
    "find_plan_create", "find_plan_destroy", "find_plan_info", "find_plan_cluster_set", "find_plan_elims",
    "find_plan_ledger", "find_ledger_key_name", "find_solve_workspace_bytes", "find_plan_upload", "find_solve",
    "find_solve_groups", "find_plan_groups", "find_solve_status", "find_solve_launch_count",
    "find_schur_sigma_update", "find_plan_exception_slots", "find_plan_specs", "find_solve_timing_enable",
    "find_solve_timing_read", "find_plan_group_phases", "find_solve_timing_read2", "find_plan_offdiag_pairs",
    "find_solve_offdiag", "find_solve_offdiag_groups", "find_plan_elim_splits", "find_plan_elim_out",
    "find_plan_arena_elems", "find_dense_create", "find_dense_destroy", "find_dense_inverse", "find_zgemm_batched",
)


class FindStatus(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("energy_idx", C.c_int32),
        ("cluster_label", C.c_int64),
        ("node_id", C.c_int64),
        ("pivot_ratio", C.c_double),
        ("message", C.c_char * 160),
    ]

    @property
    def text(self) -> str:
        return self.message.decode(errors="replace")


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(
            f"native library {LIB_PATH} is missing; build it with `python -m paper_1104_0623_b200.build`"
        )
    L = C.CDLL(str(LIB_PATH))
    P = C.c_void_p
    i32, i64, dbl, sz = C.c_int32, C.c_int64, C.c_double, C.c_size_t
    pi64, pi32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    st = C.POINTER(FindStatus)
    sig = {
        "find_plan_create": (i32, [i64, i64, pi64, pi64, i64, i32, C.POINTER(P), st]),
        "find_plan_destroy": (None, [P]),
        "find_plan_info": (i32, [P, pi64]),
        "find_plan_cluster_set": (i64, [P, i64, i32, pi64, i64]),
        "find_plan_elims": (i32, [P, pi32, pi32, pi32, pi64]),
        "find_plan_ledger": (i32, [P, i32, i32, pi64, pi64]),
        "find_ledger_key_name": (C.c_char_p, [i32]),
        "find_solve_workspace_bytes": (sz, [P, i32, i32]),
        "find_plan_upload": (i32, [P, st]),
        "find_solve": (i32, [P, P, P, i32, i32, i32, dbl, P, P, P, sz, P, st]),
        "find_solve_groups": (i32, [P, P, P, i32, i32, i32, dbl, P, P, P, sz, i64, i64, P, st]),
        "find_plan_offdiag_pairs": (i64, [P, pi64, pi64, i64]),
        "find_plan_elim_splits": (i32, [P, pi32, pi32]),
        "find_plan_elim_out": (i32, [P, pi32, pi64]),
        "find_plan_arena_elems": (i32, [P, pi64]),
        "find_solve_offdiag": (i32, [P, P, P, i32, i32, i32, dbl, P, P, P, P, P, sz, P, st]),
        "find_solve_offdiag_groups": (i32, [P, P, P, i32, i32, i32, dbl, P, P, P, P, P, sz, i64, i64, P, st]),
        "find_plan_groups": (i32, [P, pi32, pi32, pi32, pi64, pi32, pi32, pi32]),
        "find_solve_status": (i32, [P, P, i32, P, st]),
        "find_solve_launch_count": (i64, [P, i32]),
        "find_plan_exception_slots": (i64, [P, i32, pi64, i64]),
        "find_plan_specs": (i32, [P, i32, pi32, pi32, pi32, pi64]),
        "find_plan_group_phases": (i32, [P, pi32]),
        "find_solve_timing_read2": (i64, [pi32, pi32, C.POINTER(C.c_float), C.POINTER(C.c_float), i64]),
        "find_solve_timing_enable": (None, [i32]),
        "find_solve_timing_read": (i64, [pi32, pi32, C.POINTER(C.c_float), i64]),
        "find_schur_sigma_update": (i32, [i32, i32, P, P, P, P, P, P, P, P, dbl, P, P, P, i32, P, st]),
        "find_dense_create": (i32, [i32, i32, C.POINTER(P), st]),
        "find_dense_destroy": (None, [P]),
        "find_dense_inverse": (i32, [P, P, P, P, P, st]),
        "find_zgemm_batched": (i32, [i32, i32, i32, i32, P, i64, i64, P, i64, i64, i32, P, i64, i64, i32, P, st]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
