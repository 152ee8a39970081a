"""ctypes declarations of the C ABI in include/scrooge_b200.h.

The shared library is built in-tree (paper_2208_09985_b200/_lib/) by
``paper_2208_09985_b200.build``. There is no CPU fallback: if the library is
missing or a call finds no CUDA device, the call raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

LIB_PATH = _build.LIB

SG_OK, SG_INPUT, SG_CONFIG, SG_INTERNAL, SG_CUDA = 0, 1, 2, 3, 4
SG_CNT_COUNT = 7

# Every symbol include/scrooge_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "sg_abi_version", "sg_device_count", "sg_last_error", "sg_config_default",
    "sg_validate_config", "sg_align_batch", "sg_align_packed", "sg_results_free",
    "sg_cigar_string", "sg_cigar_runs", "sg_pack", "sg_packed_free",
    "sg_last_transfer_bytes", "sg_session_create", "sg_session_run", "sg_session_fetch",
    "sg_session_info", "sg_session_kernel", "sg_session_destroy", "sg_synth_packed", "sg_synth_codes",
    "sg_pairs_free", "sg_alu_peak", "sg_read_pairs", "sg_pair_file_free", "sg_write_results",
    "sg_global_align", "sg_scoring_default", "sg_score_cigar", "sg_worst_quantile", "sg_sweep",
    "sg_sweep_format", "sg_options_default", "sg_set_options", "sg_get_options",
    "sg_session_phase_cycles", "sg_session_warp_times", "sg_plan_shards",
)

SG_KERNEL = {"auto": 0, "full": 1, "mixed": 2, "wide": 3}
SG_DIAG_WARP_TIMES, SG_DIAG_PHASE_CYCLES, SG_DIAG_HOST_TRACE = 1, 2, 4


class SgConfig(C.Structure):
    _fields_ = [("W", C.c_int32), ("O", C.c_int32), ("sene", C.c_uint8), ("dent", C.c_uint8),
                ("early_termination", C.c_uint8), ("single_window", C.c_uint8),
                ("k_single", C.c_int32)]


class SgPairs(C.Structure):
    _fields_ = [("n_pairs", C.c_int64), ("text", C.c_void_p), ("text_off", C.c_void_p),
                ("text_len", C.c_void_p), ("pattern", C.c_void_p), ("pat_off", C.c_void_p),
                ("pat_len", C.c_void_p)]


class SgPackedPairs(C.Structure):
    _fields_ = [("n_pairs", C.c_int64), ("seq", C.c_void_p), ("seq_words", C.c_int64),
                ("nmask", C.c_void_p), ("text_off", C.c_void_p), ("text_len", C.c_void_p),
                ("pat_off", C.c_void_p), ("pat_len", C.c_void_p)]


class SgPairFile(C.Structure):
    _fields_ = [("n_pairs", C.c_int64), ("ids", C.POINTER(C.c_char_p)),
                ("packed", SgPackedPairs), ("_owner", C.c_void_p)]


class SgScoring(C.Structure):
    _fields_ = [("match_bonus", C.c_int32), ("mismatch_penalty", C.c_int32),
                ("gap_open", C.c_int32), ("gap_extend", C.c_int32)]


class SgSweepOptions(C.Structure):
    _fields_ = [("W_list", C.POINTER(C.c_int32)), ("n_W", C.c_int32), ("o_fixed", C.c_int32),
                ("combos", C.POINTER(C.c_uint8)), ("n_combos", C.c_int32),
                ("scoring", SgScoring), ("measure_time", C.c_int32)]


class SgSweepRow(C.Structure):
    _fields_ = [("W", C.c_int32), ("O", C.c_int32), ("sene", C.c_uint8), ("dent", C.c_uint8),
                ("et", C.c_uint8), ("q500", C.c_int64), ("q100", C.c_int64),
                ("q010", C.c_int64), ("q001", C.c_int64), ("frac_optimal", C.c_double),
                ("mean_rows_frac", C.c_double), ("stored_bits_ratio", C.c_double),
                ("pairs_per_s", C.c_double), ("oracle_q500", C.c_int64),
                ("oracle_q100", C.c_int64), ("oracle_q010", C.c_int64),
                ("oracle_q001", C.c_int64)]


class SgOptions(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("stream_upload", C.c_int32), ("longest_first", C.c_int32),
                ("diagnostics", C.c_int32), ("exact_budget", C.c_int64)]


class SgResults(C.Structure):
    _fields_ = [("n_pairs", C.c_int64), ("distance", C.POINTER(C.c_int64)),
                ("windows", C.POINTER(C.c_int32)), ("found", C.POINTER(C.c_uint8)),
                ("cigar_off", C.POINTER(C.c_int64)), ("runs", C.POINTER(C.c_uint8)),
                ("counters", C.POINTER(C.c_uint64)), ("total", C.c_uint64 * SG_CNT_COUNT),
                ("align_seconds", C.c_double), ("device_ms", C.c_double),
                ("kernel_ms", C.c_double), ("gpu_launches", C.c_int64), ("_owner", C.c_void_p)]


_lib = None


def load(build_if_missing: bool = True):
    """Loads (building first if needed) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    alt = os.environ.get("SG_LIB_OVERRIDE")  # development aid: A/B against another build
    if alt:
        build_if_missing = False
    if build_if_missing and _build._stale():
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"scrooge_b200 CUDA library missing: {LIB_PATH} "
                          "(run python -m paper_2208_09985_b200.build)")
    L = C.CDLL(alt or LIB_PATH)
    P = C.POINTER
    L.sg_abi_version.restype = C.c_int
    L.sg_device_count.restype = C.c_int
    L.sg_last_error.restype = C.c_char_p
    L.sg_config_default.argtypes = [P(SgConfig)]
    L.sg_config_default.restype = None
    L.sg_validate_config.argtypes = [P(SgConfig)]
    L.sg_align_batch.argtypes = [P(SgConfig), P(SgPairs), P(C.c_int), C.c_int, P(SgResults)]
    L.sg_align_packed.argtypes = [P(SgConfig), P(SgPackedPairs), P(C.c_int), C.c_int,
                                  P(SgResults)]
    L.sg_results_free.argtypes = [P(SgResults)]
    L.sg_results_free.restype = None
    L.sg_cigar_string.argtypes = [P(SgResults), C.c_int64, C.c_char_p, C.c_int64]
    L.sg_cigar_string.restype = C.c_int64
    L.sg_cigar_runs.argtypes = [P(SgResults), C.c_int64, C.c_char_p, P(C.c_int64), C.c_int64]
    L.sg_cigar_runs.restype = C.c_int64
    L.sg_pack.argtypes = [P(SgPairs), P(SgPackedPairs)]
    L.sg_packed_free.argtypes = [P(SgPackedPairs)]
    L.sg_packed_free.restype = None
    L.sg_last_transfer_bytes.argtypes = [C.c_int]
    L.sg_last_transfer_bytes.restype = C.c_int64
    L.sg_session_create.argtypes = [P(SgConfig), P(SgPackedPairs), C.c_int, P(C.c_void_p)]
    L.sg_session_run.argtypes = [C.c_void_p, P(C.c_float), P(C.c_float)]
    L.sg_session_fetch.argtypes = [C.c_void_p, P(SgResults)]
    L.sg_session_info.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int32), P(C.c_int32)]
    L.sg_session_kernel.argtypes = [C.c_void_p]
    L.sg_session_kernel.restype = C.c_int
    L.sg_session_destroy.argtypes = [C.c_void_p]
    L.sg_session_destroy.restype = None
    L.sg_synth_packed.argtypes = [C.c_int, C.c_int64, C.c_int64, P(SgPackedPairs)]
    L.sg_synth_codes.argtypes = [C.c_int, C.c_int64, C.c_int64, P(SgPairs)]
    L.sg_pairs_free.argtypes = [P(SgPairs)]
    L.sg_pairs_free.restype = None
    L.sg_alu_peak.argtypes = [C.c_int, P(C.c_double), P(C.c_double), P(C.c_double)]
    L.sg_read_pairs.argtypes = [C.c_char_p, C.c_int, P(SgPairFile)]
    L.sg_pair_file_free.argtypes = [P(SgPairFile)]
    L.sg_pair_file_free.restype = None
    L.sg_write_results.argtypes = [C.c_char_p, P(SgPairFile), P(SgResults), C.c_int]
    L.sg_global_align.argtypes = [P(SgPackedPairs), C.c_int, P(SgResults)]
    L.sg_scoring_default.argtypes = [P(SgScoring)]
    L.sg_scoring_default.restype = None
    L.sg_score_cigar.argtypes = [P(SgResults), C.c_int64, P(SgScoring)]
    L.sg_score_cigar.restype = C.c_int64
    L.sg_worst_quantile.argtypes = [P(C.c_int64), C.c_int64, C.c_double, P(C.c_int64)]
    L.sg_sweep.argtypes = [P(SgSweepOptions), P(SgPackedPairs), P(C.c_int), C.c_int, P(SgSweepRow)]
    L.sg_sweep_format.argtypes = [P(SgSweepRow), C.c_int64, C.c_int, C.c_char_p, C.c_int64]
    L.sg_sweep_format.restype = C.c_int64
    L.sg_options_default.argtypes = [P(SgOptions)]
    L.sg_options_default.restype = None
    L.sg_set_options.argtypes = [P(SgOptions)]
    L.sg_get_options.argtypes = [P(SgOptions)]
    L.sg_get_options.restype = None
    L.sg_session_phase_cycles.argtypes = [C.c_void_p, P(C.c_uint64)]
    L.sg_session_warp_times.argtypes = [C.c_void_p, P(C.c_uint64), C.c_int]
    L.sg_plan_shards.argtypes = [P(SgPackedPairs), C.c_int, C.c_void_p, C.c_void_p, P(C.c_int)]
    _lib = L
    return L


def last_error() -> str:
    return load().sg_last_error().decode(errors="replace")
