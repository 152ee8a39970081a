"""ctypes bindings for the C oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: the oracle is the CPU checker the GPU path is
compared against. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB_PATH = os.path.join(ORACLE_DIR, "_build", "liboracle.so")
REF_TOOL = os.path.join(ORACLE_DIR, "_ref", "ref_tool")


class OrcConfig(C.Structure):
    _fields_ = [("W", C.c_int32), ("O", C.c_int32), ("sene", C.c_uint8), ("dent", C.c_uint8),
                ("et", C.c_uint8), ("single_window", C.c_uint8), ("k_single", C.c_int32)]


class OrcCounters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "stored_bits", "table_writes", "table_reads", "rows_computed", "cells_computed",
        "rows_possible", "baseline_equiv_bits")]


class OrcResult(C.Structure):
    _fields_ = [("found", C.c_int32), ("distance", C.c_int64), ("windows", C.c_int32),
                ("n_runs", C.c_int64), ("ops", C.POINTER(C.c_char)),
                ("lens", C.POINTER(C.c_int64)), ("counters", OrcCounters)]


class SynthSpec(C.Structure):
    _fields_ = [("n_pairs", C.c_int64), ("seed", C.c_uint64), ("read_min", C.c_int32),
                ("read_max", C.c_int32), ("slack_abs", C.c_int32), ("slack_frac", C.c_double),
                ("rate_min", C.c_double), ("rate_max", C.c_double), ("mix_sub", C.c_double),
                ("mix_ins", C.c_double), ("mix_del", C.c_double),
                ("frac_uncorrelated", C.c_double)]


_lib = None


def ensure_built() -> None:
    src = [os.path.join(ORACLE_DIR, f) for f in ("genasm_oracle.c", "genasm_oracle.h")]
    if not os.path.exists(LIB_PATH) or any(os.path.getmtime(f) > os.path.getmtime(LIB_PATH)
                                           for f in src):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "all"], check=True)


def lib():
    global _lib
    if _lib is None:
        ensure_built()
        L = C.CDLL(LIB_PATH)
        L.orc_align.argtypes = [C.POINTER(OrcConfig), C.c_char_p, C.c_int64, C.c_char_p,
                                C.c_int64, C.POINTER(OrcResult), C.c_char_p, C.c_size_t]
        L.orc_align.restype = C.c_int
        L.orc_result_free.argtypes = [C.POINTER(OrcResult)]
        L.orc_last_window_count.restype = C.c_int64
        L.orc_last_window_stats.argtypes = [C.POINTER(C.c_int32)] * 3 + [C.c_int64]
        L.sg_synth_baseline_spec.argtypes = [C.c_int, C.POINTER(SynthSpec)]
        L.sg_synth_max_text.argtypes = [C.POINTER(SynthSpec)]
        L.sg_synth_max_text.restype = C.c_int64
        L.sg_synth_max_pattern.argtypes = [C.POINTER(SynthSpec)]
        L.sg_synth_max_pattern.restype = C.c_int64
        L.sg_synth_pair.argtypes = [C.POINTER(SynthSpec), C.c_int64, C.c_char_p,
                                    C.POINTER(C.c_int64), C.c_char_p, C.POINTER(C.c_int64)]
        L.orc_replay_runs.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, C.c_void_p,
                                      C.c_int64]
        L.orc_replay_runs.restype = C.c_int64
        L.orc_replay_batch.argtypes = [C.c_int64] + [C.c_void_p] * 9 + [C.c_int]
        L.orc_replay_batch.restype = C.c_int64
        L.orc_global_align.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64,
                                       C.POINTER(OrcResult), C.c_char_p, C.c_size_t]
        L.orc_score_cigar.argtypes = [C.POINTER(OrcResult)] + [C.c_int] * 4
        L.orc_score_cigar.restype = C.c_int64
        L.orc_worst_quantile.argtypes = [C.POINTER(C.c_int64), C.c_int64, C.c_double]
        L.orc_worst_quantile.restype = C.c_int64
        L.orc_digest_blocks.argtypes = [C.c_int64] + [C.c_void_p] * 6 + [C.c_int64, C.c_void_p,
                                                                          C.c_int]
        L.orc_digest_blocks.restype = C.c_uint64
        _lib = L
    return _lib


COUNTER_NAMES = [n for n, _ in OrcCounters._fields_]


@dataclass
class Alignment:
    found: bool
    distance: int
    cigar: str
    windows: int
    counters: dict = field(default_factory=dict)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def align(text: bytes, pattern: bytes, W=64, O=33, sene=True, dent=True, et=True,
          single_window=False, k_single=1024) -> Alignment:
    """Oracle align() on 1-byte base codes (0..3 ACGT, 4 other)."""
    L = lib()
    cfg = OrcConfig(W, O, int(sene), int(dent), int(et), int(single_window), k_single)
    res = OrcResult()
    err = C.create_string_buffer(512)
    rc = L.orc_align(C.byref(cfg), bytes(text), len(text), bytes(pattern), len(pattern),
                     C.byref(res), err, len(err))
    if rc:
        raise OracleError(rc, err.value.decode())
    cig = "".join(f"{res.lens[k]}{res.ops[k].decode()}" for k in range(res.n_runs))
    out = Alignment(bool(res.found), res.distance, cig if res.found else "*", res.windows,
                    {n: getattr(res.counters, n) for n in COUNTER_NAMES})
    L.orc_result_free(C.byref(res))
    return out


def global_align(text: bytes, pattern: bytes, scoring=(2, 4, 4, 2)):
    """Oracle global_align (proj/src/oracle.cpp:39-89) -> (distance, cigar, score_cigar)."""
    L = lib()
    res = OrcResult()
    err = C.create_string_buffer(512)
    rc = L.orc_global_align(bytes(text), len(text), bytes(pattern), len(pattern), C.byref(res),
                            err, len(err))
    if rc:
        raise OracleError(rc, err.value.decode())
    cig = "".join(f"{res.lens[k]}{res.ops[k].decode()}" for k in range(res.n_runs))
    score = L.orc_score_cigar(C.byref(res), *scoring)
    out = (res.distance, cig, score)
    L.orc_result_free(C.byref(res))
    return out


def worst_quantile(scores, p: float) -> int:
    """worst_quantile (proj/src/sweep.cpp:11-19)."""
    arr = (C.c_int64 * len(scores))(*scores)
    return lib().orc_worst_quantile(arr, len(scores), p)


def window_stats():
    """(d_opt, n_w, m_w) of every window of the last align() on this thread."""
    L = lib()
    n = L.orc_last_window_count()
    a = (C.c_int32 * n)()
    b = (C.c_int32 * n)()
    c = (C.c_int32 * n)()
    L.orc_last_window_stats(a, b, c, n)
    return list(a), list(b), list(c)


def baseline_spec(cfg_id: int) -> SynthSpec:
    s = SynthSpec()
    if not lib().sg_synth_baseline_spec(cfg_id, C.byref(s)):
        raise ValueError(cfg_id)
    return s


def synth_pair(spec: SynthSpec, p: int):
    L = lib()
    tb = C.create_string_buffer(L.sg_synth_max_text(C.byref(spec)))
    pb = C.create_string_buffer(L.sg_synth_max_pattern(C.byref(spec)))
    n = C.c_int64()
    m = C.c_int64()
    L.sg_synth_pair(C.byref(spec), p, tb, C.byref(n), pb, C.byref(m))
    return tb.raw[:n.value], pb.raw[:m.value]


def encode(s: str) -> bytes:
    """encode_sequence, proj/include/scrooge/sequence.hpp:19-37."""
    tbl = {"A": 0, "C": 1, "G": 2, "T": 3, "a": 0, "c": 1, "g": 2, "t": 3}
    return bytes(tbl.get(ch, 4) for ch in s)


def decode(b: bytes) -> str:
    return "".join("ACGTN"[min(x, 4)] for x in b)


def fnv1a(s: str) -> str:
    h = 1469598103934665603
    for ch in s.encode():
        h = ((h ^ ch) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def replay_batch(codes, results, threads=None) -> int:
    """Pairs of a CodesBatch whose GPU CIGAR fails validate_replay or whose edit
    count differs from the reported distance (proj/src/cigar.cpp:70-107)."""
    import numpy as np
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    dist = np.ascontiguousarray(results.distance, dtype=np.int64)
    return int(lib().orc_replay_batch(codes.n, ptr(codes.text), ptr(codes.text_off),
                                      ptr(codes.text_len), ptr(codes.pattern), ptr(codes.pat_off),
                                      ptr(codes.pat_len), ptr(results.runs),
                                      ptr(results.cigar_off), ptr(dist),
                                      threads or (os.cpu_count() or 8)))


def digest_blocks(distance, windows, found, cigar_off, runs, counters, block=1000, threads=None):
    """Per-block digests of a batch's results (orc_digest_blocks; the same records as
    `ref_tool digest`, oracle/ref_tool.cpp:digest_line) -> (list of hex, total hex)."""
    import numpy as np
    n = len(distance)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    dist = np.ascontiguousarray(distance, dtype=np.int64)
    win = np.ascontiguousarray(windows, dtype=np.int32)
    fnd = None if found is None else np.ascontiguousarray(found, dtype=np.uint8)
    off = np.ascontiguousarray(cigar_off, dtype=np.int64)
    rb = np.ascontiguousarray(runs, dtype=np.uint8)
    if rb.size == 0:
        rb = np.zeros(1, np.uint8)
    cnt = np.ascontiguousarray(counters, dtype=np.uint64).reshape(-1)
    out = np.zeros(max(1, (n + block - 1) // block), np.uint64)
    total = lib().orc_digest_blocks(n, ptr(dist), ptr(win), None if fnd is None else ptr(fnd),
                                    ptr(off), ptr(rb), ptr(cnt), block, ptr(out),
                                    threads or os.cpu_count() or 8)
    return [f"{int(x):016x}" for x in out[: (n + block - 1) // block]], f"{total:016x}"


def results_digests(res, block=1000):
    """digest_blocks over a paper_2208_09985_b200 Results object."""
    return digest_blocks(res.distance, res.windows, res.found, res.cigar_off, res.runs,
                         res.counters, block)


def runs_from_cigar(cigar: str) -> bytes:
    """The GPU path's run-byte encoding ((op << 6) | (len - 1), <= 64 per byte) of a
    CIGAR string; used to pin the digest over run bytes without a GPU."""
    import re
    out = bytearray()
    for n, op in re.findall(r"(\d+)([=XID])", cigar):
        n = int(n)
        code = "=XID".index(op)
        while n > 0:
            k = min(n, 64)
            out.append((code << 6) | (k - 1))
            n -= k
    return bytes(out)
