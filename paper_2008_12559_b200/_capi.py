"""ctypes binding of include/pft_capi.h (the C ABI of libpft_b200.so).

This module only declares signatures; the user-facing mirror of the reference's
plan/execute interface lives in paper_2008_12559_b200/__init__.py.  Loading fails
loudly when the shared library is missing -- there is no pure-Python fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libpft_b200.so"


class c128(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class PlanInfo(C.Structure):
    _fields_ = [("N", C.c_uint64), ("M", C.c_uint64), ("mu", C.c_int64), ("p", C.c_uint64),
                ("q", C.c_uint64), ("r", C.c_int32), ("reserved", C.c_int32), ("epsilon", C.c_double),
                ("achieved_epsilon", C.c_double), ("xi", C.c_double), ("estimated_cost", C.c_double),
                ("plan_id", C.c_uint64)]


class DPlanOpts(C.Structure):
    _fields_ = [("device", C.c_int), ("p2", C.c_uint64), ("k1_stages", C.c_int), ("second_pass", C.c_int),
                ("k2_at", C.c_int), ("tail_ctas", C.c_int), ("k2_grid_ctas", C.c_int), ("k1_split", C.c_int),
                ("reserved", C.c_int),
                ("batch_hint", C.c_uint64)]


class ShardInfo(C.Structure):
    _fields_ = [("pair_begin", C.c_uint64), ("pair_end", C.c_uint64), ("row_len", C.c_uint64),
                ("front_col", C.c_int64), ("mirror_col", C.c_int64), ("single0_col", C.c_int64),
                ("singleh_col", C.c_int64)]


class SignalDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("seed", C.c_uint64), ("N", C.c_uint64), ("index_offset", C.c_uint64),
                ("n_tones", C.c_int), ("freqs", C.POINTER(C.c_int64)), ("amps", C.POINTER(c128)),
                ("sigma", C.c_double)]


P = C.c_void_p
D = C.c_double
U64 = C.c_uint64
I64 = C.c_int64
SZ = C.c_size_t
I = C.c_int
ST = C.c_int  # pft_status
PC = C.POINTER(c128)
PD = C.POINTER(C.c_double)

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "pft_status_string": (C.c_char_p, [ST]),
    "pft_last_error": (C.c_char_p, []),
    "pft_version": (C.c_char_p, []),
    "pft_best_approx": (ST, [I, D, D, P, PD]),
    "pft_scope_xi": (ST, [D, I, PD, P, PD]),
    "pft_translate_poly": (ST, [P, I, D, D, P]),
    "pft_table_default": (ST, [C.POINTER(P)]),
    "pft_table_generate": (ST, [P, I, I, C.POINTER(P)]),
    "pft_table_save": (ST, [P, C.c_char_p]),
    "pft_table_load": (ST, [C.c_char_p, C.POINTER(P)]),
    "pft_table_save_csv": (ST, [P, C.c_char_p]),
    "pft_table_destroy": (None, [P]),
    "pft_table_size": (ST, [P, C.POINTER(SZ)]),
    "pft_table_entry": (ST, [P, SZ, PD, C.POINTER(I), PD, P, PD]),
    "pft_table_lookup": (ST, [P, D, I, PD, P, PD]),
    "pft_divisors": (ST, [U64, P, SZ, C.POINTER(SZ)]),
    "pft_min_terms": (ST, [P, D, U64, U64, C.POINTER(I)]),
    "pft_select_divisor": (ST, [P, U64, U64, D, C.POINTER(U64), C.POINTER(I), PD]),
    "pft_select_divisor_device": (ST, [P, U64, U64, D, I, C.POINTER(U64), C.POINTER(I), PD]),
    "pft_workspace_bytes_2d": (ST, [P, P, C.POINTER(SZ)]),
    "pft_execute_2d": (ST, [P, P, P, P, P, P]),
    "pft_execute_2d_host": (ST, [P, P, P, P]),
    "pft_autotune_divisor": (ST, [P, U64, U64, I64, D, I, P, SZ, I, C.POINTER(U64), PD]),
    "pft_plan_build": (ST, [P, U64, U64, I64, U64, D, C.POINTER(P)]),
    "pft_plan_destroy": (None, [P]),
    "pft_plan_info_get": (ST, [P, C.POINTER(PlanInfo)]),
    "pft_plan_copy_B": (ST, [P, P]),
    "pft_plan_copy_w": (ST, [P, P]),
    "pft_plan_copy_phase": (ST, [P, P]),
    "pft_plan_copy_tvals": (ST, [P, P]),
    "pft_plan_copy_post_powers": (ST, [P, P]),
    "pft_plan_copy_post_twiddles": (ST, [P, P]),
    "pft_plan_json": (ST, [P, C.c_char_p, SZ, C.POINTER(SZ)]),
    "pft_dplan_create": (ST, [P, C.POINTER(DPlanOpts), C.POINTER(P)]),
    "pft_dplan_destroy": (None, [P]),
    "pft_dplan_layout": (ST, [P, C.POINTER(U64), C.POINTER(U64)]),
    "pft_workspace_bytes": (ST, [P, SZ, C.POINTER(SZ)]),
    "pft_partial_bytes": (ST, [P, SZ, C.POINTER(SZ)]),
    "pft_execute": (ST, [P, P, SZ, SZ, P, P, P]),
    "pft_execute_ex": (ST, [P, P, SZ, SZ, P, P, P, C.c_uint]),
    "pft_workspace_status": (ST, [P, P, P, C.POINTER(I), I]),
    "pft_execute_partial": (ST, [P, P, I, I, U64, P, P]),
    "pft_finalize": (ST, [P, P, SZ, P, P]),
    "pft_shard_layout": (ST, [U64, I, I, C.POINTER(ShardInfo)]),
    "pft_shard_gather_host": (ST, [U64, U64, I, I, P, P, U64]),
    "pft_status_query": (ST, [P, P, C.POINTER(I), I]),
    "pft_execute_host": (ST, [P, P, SZ, P, P, P, P]),
    "pft_generate_host": (ST, [C.POINTER(SignalDesc), P, U64]),
    "pft_generate_device": (ST, [C.POINTER(SignalDesc), P, U64, P]),
    "pft_sparse_tones": (ST, [U64, I, I64, I64, P, P]),
    "pft_launches_per_execute": (ST, [P, C.POINTER(I)]),
    "pft_dplan_signals_per_cta": (ST, [P, SZ, C.POINTER(I)]),
    "pft_dplan_tail_kind": (ST, [P, C.POINTER(I)]),
    "pft_dplan_second_pass": (ST, [P, C.POINTER(I)]),
    "pft_naive_dft_device": (ST, [P, U64, I64, U64, P, P]),
    "pft_naive_dft_host": (ST, [P, U64, I64, U64, P]),
    "pft_device_count": (ST, [C.POINTER(I)]),
    "pft_signal_read": (ST, [C.c_char_p, I, P, U64, C.POINTER(U64), C.POINTER(I)]),
    "pft_signal_write": (ST, [C.c_char_p, I, P, U64, I]),
    "pft_spectrum_write_csv": (ST, [C.c_char_p, I64, U64, P]),
    "pft_spectrum_read_csv": (ST, [C.c_char_p, C.POINTER(I64), P, U64, C.POINTER(U64)]),
    "pft_anomaly_from_coeffs": (ST, [P, U64, P, U64, U64, P, P, P]),
    "pft_anomaly": (ST, [P, P, U64, P, P, P]),
    "pft_dplan_shape": (ST, [P, C.POINTER(U64), C.POINTER(U64), C.POINTER(I64)]),
    "pft_dplan_device": (ST, [P, C.POINTER(I)]),
    "pft_nccl_available": (ST, [C.POINTER(I)]),
    "pft_nccl_get_unique_id": (ST, [P]),
    "pft_nccl_comm_init": (ST, [I, I, P, I, C.POINTER(P)]),
    "pft_nccl_comm_destroy": (ST, [P]),
    "pft_execute_sharded": (ST, [P, P, U64, P, I, P, P, P]),
    "pft_select_divisor_sharded": (ST, [P, U64, U64, D, I, I, C.POINTER(U64), C.POINTER(I), PD]),
}

STATUS_NAMES = {
    0: "PFT_OK", 1: "PFT_ERR_INVALID_ARGUMENT", 2: "PFT_ERR_P_NOT_DIVISOR", 3: "PFT_ERR_M_TOO_LARGE",
    4: "PFT_ERR_EPSILON_NOT_IN_TABLE", 5: "PFT_ERR_RATIO_OUT_OF_RANGE", 6: "PFT_ERR_LENGTH_MISMATCH",
    7: "PFT_ERR_NON_FINITE", 8: "PFT_ERR_IO", 9: "PFT_ERR_VERSION_MISMATCH", 10: "PFT_ERR_NO_DEVICE",
    11: "PFT_ERR_CUDA", 12: "PFT_ERR_UNSUPPORTED", 13: "PFT_ERR_INTERNAL", 14: "PFT_ERR_BUFFER_TOO_SMALL",
}

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load libpft_b200.so (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("PFT_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(f"{path} not found: build it with `python -m paper_2008_12559_b200.build` "
                          "(there is no pure-Python fallback)")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:  # an older development build (PFT_LIB) without this entry point
            if path == LIB_PATH:
                raise ImportError(f"{path} does not export {name}: rebuild it")
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
