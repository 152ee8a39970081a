"""Python mirror of the reference aligner API over the sm_100a C ABI.

Names, argument meaning and error behaviour follow the reference's
``proj/include/scrooge/`` so code (and tests) written against the reference
read the same way here:

=========================  ==========================================================
reference                  here
=========================  ==========================================================
AlignerConfig              :class:`AlignerConfig` (aligner.hpp:12-31)
InstrumentationCounters    :class:`InstrumentationCounters` (dp.hpp:46-66)
AlignmentResult / align    :class:`AlignmentResult`, :func:`align` (aligner.hpp:33-45)
PairOutcome / BatchResult  :class:`PairOutcome`, :class:`BatchResult` (batch.hpp:14-27)
run_batch                  :func:`run_batch` (batch.hpp:33-34, batch.cpp:13-104)
write_batch_tsv            :func:`write_batch_tsv` (batch.cpp:106-113)
SeqPairRecord              :class:`SeqPairRecord` (io.hpp:9-13)
encode_sequence            :func:`encode_sequence` (sequence.hpp:19-37)
cigar_to_string            :func:`cigar_to_string` (cigar.cpp:18-25)
InputError / ConfigError   :class:`InputError` / :class:`ConfigError` (errors.hpp:10-20)
InternalError              :class:`InternalError` (errors.hpp:24-34)
=========================  ==========================================================

Everything that computes runs on the GPU through ``libscrooge_b200.so``; there
is no CPU fallback.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import re
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np

from . import _ffi
from ._ffi import SG_CONFIG, SG_CUDA, SG_INPUT, SG_INTERNAL, SG_OK


# ----------------------------------------------------------------- errors

class InputError(Exception):
    """scrooge::InputError (proj/include/scrooge/errors.hpp:10-13)."""


class ConfigError(Exception):
    """scrooge::ConfigError (errors.hpp:17-20)."""


class InternalError(Exception):
    """scrooge::InternalError (errors.hpp:24-27)."""


class OutOfStoredRegionError(InternalError):
    """scrooge::OutOfStoredRegionError (errors.hpp:31-34)."""


class CudaError(RuntimeError):
    """Device or driver failure (no reference equivalent; never a CPU fallback)."""


_ERRORS = {SG_INPUT: InputError, SG_CONFIG: ConfigError, SG_INTERNAL: InternalError,
           SG_CUDA: CudaError}


def _raise(rc: int, ids: Optional[Sequence[str]] = None):
    msg = _ffi.last_error()
    if ids is not None:
        m = re.match(r"pair '(\d+)': (.*)", msg)
        if m and int(m.group(1)) < len(ids):
            msg = f"pair '{ids[int(m.group(1))]}': {m.group(2)}"
    raise _ERRORS.get(rc, CudaError)(msg)


def _check(rc: int, ids=None):
    if rc != SG_OK:
        _raise(rc, ids)


# ----------------------------------------------------------------- config / results

@dataclass
class AlignerConfig:
    """AlignerConfig (proj/include/scrooge/aligner.hpp:12-31)."""
    W: int = 64
    O: int = 33
    sene: bool = True
    dent: bool = True
    early_termination: bool = True
    mode: str = "windowed"  # "windowed" | "single"
    k_single: int = 1024

    def _c(self) -> _ffi.SgConfig:
        return _ffi.SgConfig(int(self.W), int(self.O), int(bool(self.sene)), int(bool(self.dent)),
                             int(bool(self.early_termination)), int(self.mode == "single"),
                             int(self.k_single))

    def validate(self) -> None:
        """AlignerConfig::validate (aligner.cpp:8-18) plus the GPU path's limits."""
        if self.mode not in ("windowed", "single"):
            raise ConfigError(f"unknown mode '{self.mode}'")
        _check(_ffi.load().sg_validate_config(C.byref(self._c())))

    def storage_policy(self) -> str:
        """aligner.hpp:26-30."""
        if self.dent:
            return "DentTrimmed"
        if self.sene:
            return "SeneEntries"
        return "BaselineEdges"


_COUNTER_NAMES = ("stored_bits", "table_writes", "table_reads", "rows_computed",
                  "cells_computed", "rows_possible", "baseline_equiv_bits")


@dataclass
class InstrumentationCounters:
    """InstrumentationCounters (proj/include/scrooge/dp.hpp:46-66)."""
    stored_bits: int = 0
    table_writes: int = 0
    table_reads: int = 0
    rows_computed: int = 0
    cells_computed: int = 0
    rows_possible: int = 0
    baseline_equiv_bits: int = 0

    def add(self, o: "InstrumentationCounters") -> None:
        for n in _COUNTER_NAMES:
            setattr(self, n, getattr(self, n) + getattr(o, n))

    @classmethod
    def from_array(cls, a) -> "InstrumentationCounters":
        return cls(*(int(x) for x in a))


Cigar = list  # list[tuple[str, int]] — CigarOp{op, len} (cigar.hpp:15-21)


def cigar_to_string(cigar: Iterable) -> str:
    """cigar_to_string (proj/src/cigar.cpp:18-25)."""
    return "".join(f"{n}{op}" for op, n in cigar)


def cigar_from_string(s: str) -> Cigar:
    """cigar_from_string (proj/src/cigar.cpp:27-47)."""
    out: Cigar = []
    pos = 0
    while pos < len(s):
        m = re.match(r"(\d+)([=XID])", s[pos:])
        if not m:
            raise InputError(f"malformed CIGAR at position {pos}")
        n = int(m.group(1))
        if n == 0:
            raise InputError("malformed CIGAR: zero-length run")
        if out and out[-1][0] == m.group(2):
            out[-1] = (out[-1][0], out[-1][1] + n)
        else:
            out.append((m.group(2), n))
        pos += m.end()
    return out


@dataclass
class AlignmentResult:
    """AlignmentResult (aligner.hpp:33-38)."""
    distance: int = 0
    cigar: Cigar = field(default_factory=list)
    windows: int = 0
    counters: InstrumentationCounters = field(default_factory=InstrumentationCounters)


@dataclass
class PairOutcome:
    """PairOutcome (batch.hpp:14-20)."""
    found: bool = True
    distance: int = -1
    cigar: Cigar = field(default_factory=list)
    windows: int = 0
    counters: InstrumentationCounters = field(default_factory=InstrumentationCounters)


@dataclass
class BatchResult:
    """BatchResult (batch.hpp:22-27) + device timings of the GPU run."""
    outcomes: list = field(default_factory=list)
    total: InstrumentationCounters = field(default_factory=InstrumentationCounters)
    align_seconds: float = 0.0
    pairs_per_second: float = 0.0
    device_ms: float = 0.0
    kernel_ms: float = 0.0
    gpu_launches: int = 0


@dataclass
class SeqPairRecord:
    """SeqPairRecord (io.hpp:9-13)."""
    id: str
    text: str
    pattern: str


# ----------------------------------------------------------------- sequences

_ENC = np.full(256, 4, dtype=np.uint8)
for _c, _v in zip(b"ACGTacgt", (0, 1, 2, 3, 0, 1, 2, 3)):
    _ENC[_c] = _v


def encode_sequence(s) -> bytes:
    """encode_sequence (sequence.hpp:33-37): A,C,G,T -> 0..3, anything else -> 4."""
    if isinstance(s, (bytes, bytearray, memoryview, np.ndarray)):
        return bytes(s)
    return _ENC[np.frombuffer(s.encode("latin-1"), dtype=np.uint8)].tobytes()


def decode_sequence(codes: bytes) -> str:
    return "".join("ACGTN"[min(c, 4)] for c in codes)


# ----------------------------------------------------------------- raw batches

class Results:
    """Owned sg_results: numpy views of distances, windows, counters and runs."""

    _OPS = "=XID"

    def __init__(self, res: _ffi.SgResults):
        self._res = res
        n = res.n_pairs
        self.n = n
        self.distance = np.ctypeslib.as_array(res.distance, (max(n, 1),))[:n]
        self.windows = np.ctypeslib.as_array(res.windows, (max(n, 1),))[:n]
        self.found = np.ctypeslib.as_array(res.found, (max(n, 1),))[:n]
        self.cigar_off = np.ctypeslib.as_array(res.cigar_off, (n + 1,))
        nb = int(self.cigar_off[n]) if n else 0
        self.runs = np.ctypeslib.as_array(res.runs, (max(nb, 1),))[:nb]
        self.counters = np.ctypeslib.as_array(res.counters, (max(n, 1) * 7,)).reshape(-1, 7)[:n]
        self.total = InstrumentationCounters.from_array(res.total)
        self.align_seconds = res.align_seconds
        self.device_ms = res.device_ms
        self.kernel_ms = res.kernel_ms
        self.gpu_launches = res.gpu_launches

    def __del__(self):
        try:
            _ffi.load().sg_results_free(C.byref(self._res))
        except Exception:
            pass

    def cigar(self, k: int) -> Cigar:
        lo, hi = int(self.cigar_off[k]), int(self.cigar_off[k + 1])
        out: Cigar = []
        for b in self.runs[lo:hi].tolist():
            op, n = self._OPS[b >> 6], (b & 63) + 1
            if out and out[-1][0] == op:
                out[-1] = (op, out[-1][1] + n)
            else:
                out.append((op, n))
        return out

    def cigar_string(self, k: int) -> str:
        L = _ffi.load()
        need = L.sg_cigar_string(C.byref(self._res), k, None, 0)
        buf = C.create_string_buffer(int(need) + 1)
        L.sg_cigar_string(C.byref(self._res), k, buf, len(buf))
        return buf.value.decode()

    def pair_counters(self, k: int) -> InstrumentationCounters:
        return InstrumentationCounters.from_array(self.counters[k])


class PackedBatch:
    """Owned 2-bit packed pairs (sg_packed_pairs)."""

    def __init__(self, p: _ffi.SgPackedPairs):
        self._p = p
        self.n = p.n_pairs

    @property
    def c(self) -> _ffi.SgPackedPairs:
        return self._p

    def lengths(self):
        n = self.n
        tl = np.ctypeslib.as_array(C.cast(self._p.text_len, C.POINTER(C.c_int64)), (max(n, 1),))[:n]
        pl = np.ctypeslib.as_array(C.cast(self._p.pat_len, C.POINTER(C.c_int64)), (max(n, 1),))[:n]
        return tl, pl

    def input_bytes(self) -> int:
        """Bytes of packed sequence words (the H2D payload's bulk)."""
        return 4 * int(self._p.seq_words)

    def __del__(self):
        try:
            _ffi.load().sg_packed_free(C.byref(self._p))
        except Exception:
            pass


class CodesBatch:
    """1-byte-code pairs with numpy storage (keeps the arrays alive)."""

    def __init__(self, text: np.ndarray, text_off, text_len, pattern: np.ndarray, pat_off,
                 pat_len, owner: Optional[_ffi.SgPairs] = None):
        self.text = np.ascontiguousarray(text, dtype=np.uint8)
        self.pattern = np.ascontiguousarray(pattern, dtype=np.uint8)
        self.text_off = np.ascontiguousarray(text_off, dtype=np.int64)
        self.text_len = np.ascontiguousarray(text_len, dtype=np.int64)
        self.pat_off = np.ascontiguousarray(pat_off, dtype=np.int64)
        self.pat_len = np.ascontiguousarray(pat_len, dtype=np.int64)
        self.n = len(self.text_len)
        self._owner = owner

    @classmethod
    def from_lists(cls, texts: Sequence[bytes], patterns: Sequence[bytes]) -> "CodesBatch":
        tl = np.array([len(t) for t in texts], dtype=np.int64)
        pl = np.array([len(p) for p in patterns], dtype=np.int64)
        to = np.concatenate([[0], np.cumsum(tl)[:-1]]) if len(tl) else np.zeros(0, np.int64)
        po = np.concatenate([[0], np.cumsum(pl)[:-1]]) if len(pl) else np.zeros(0, np.int64)
        t = np.frombuffer(b"".join(bytes(x) for x in texts) or b"\0", dtype=np.uint8)
        p = np.frombuffer(b"".join(bytes(x) for x in patterns) or b"\0", dtype=np.uint8)
        return cls(t, to, tl, p, po, pl)

    def c(self) -> _ffi.SgPairs:
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)
        return _ffi.SgPairs(self.n, ptr(self.text), ptr(self.text_off), ptr(self.text_len),
                            ptr(self.pattern), ptr(self.pat_off), ptr(self.pat_len))

    def pair(self, k: int):
        t = self.text[self.text_off[k]:self.text_off[k] + self.text_len[k]].tobytes()
        p = self.pattern[self.pat_off[k]:self.pat_off[k] + self.pat_len[k]].tobytes()
        return t, p

    def __del__(self):
        if self._owner is not None:
            try:
                _ffi.load().sg_pairs_free(C.byref(self._owner))
            except Exception:
                pass


def _devices(devices):
    if devices is None:
        return None, 0
    arr = (C.c_int * len(devices))(*devices)
    return arr, len(devices)


def align_codes(config: AlignerConfig, batch: CodesBatch, devices=None, ids=None) -> Results:
    """run_batch core over 1-byte codes (host packing + H2D + K1-K3 + D2H)."""
    L = _ffi.load()
    res = _ffi.SgResults()
    darr, nd = _devices(devices)
    c = batch.c()
    _check(L.sg_align_batch(C.byref(config._c()), C.byref(c), darr, nd, C.byref(res)), ids)
    return Results(res)


def align_packed(config: AlignerConfig, batch: PackedBatch, devices=None) -> Results:
    """run_batch core over 2-bit packed host buffers (H2D + K1-K3 + D2H)."""
    L = _ffi.load()
    res = _ffi.SgResults()
    darr, nd = _devices(devices)
    _check(L.sg_align_packed(C.byref(config._c()), C.byref(batch.c), darr, nd, C.byref(res)))
    return Results(res)


def pack(batch: CodesBatch) -> PackedBatch:
    out = _ffi.SgPackedPairs()
    _check(_ffi.load().sg_pack(C.byref(batch.c()), C.byref(out)))
    return PackedBatch(out)


class PairFile:
    """Pairs read from a TSV or FASTA-pair file (sg_read_pairs; io.cpp:66-121),
    already 2-bit packed. `.packed` goes to align_packed; `.ids` are the pair ids."""

    def __init__(self, f: _ffi.SgPairFile):
        self._f = f
        self.n = int(f.n_pairs)
        self.ids = [f.ids[k].decode() for k in range(self.n)]
        self.packed = _PackedView(f.packed, self)

    def codes(self, k: int):
        """(text, pattern) of pair k as 1-byte codes (0..3 ACGT, 4 other)."""
        return _unpack(self._f.packed, k)

    def __del__(self):
        try:
            _ffi.load().sg_pair_file_free(C.byref(self._f))
        except Exception:
            pass


class _PackedView:
    """Non-owning view of packed pairs held by another object."""

    def __init__(self, p: _ffi.SgPackedPairs, owner):
        self._p, self._owner, self.n = p, owner, p.n_pairs

    @property
    def c(self) -> _ffi.SgPackedPairs:
        return self._p


def _unpack(p: _ffi.SgPackedPairs, k: int):
    def one(off_ptr, len_ptr):
        off = C.cast(off_ptr, C.POINTER(C.c_int64))[k]
        n = C.cast(len_ptr, C.POINTER(C.c_int64))[k]
        idx = np.arange(off, off + n, dtype=np.int64)
        words = np.ctypeslib.as_array(C.cast(p.seq, C.POINTER(C.c_uint32)), (int(p.seq_words),))
        codes = ((words[idx >> 4] >> (2 * (idx & 15)).astype(np.uint32)) & 3).astype(np.uint8)
        if p.nmask:
            nw = (int(p.seq_words) * 16 + 31) // 32
            nm = np.ctypeslib.as_array(C.cast(p.nmask, C.POINTER(C.c_uint32)), (nw,))
            codes[((nm[idx >> 5] >> (idx & 31).astype(np.uint32)) & 1) == 1] = 4
        return codes.tobytes()
    return one(p.text_off, p.text_len), one(p.pat_off, p.pat_len)


def read_pairs(path: str, fmt: str = "tsv") -> PairFile:
    """read_pairs (proj/src/io.cpp:114-121): fmt "tsv" or "fasta-pair"
    (path = "<text.fa>,<pattern.fa>")."""
    if fmt not in ("tsv", "fasta-pair"):
        raise InputError(f"unknown input format '{fmt}' (expected tsv or fasta-pair)")
    out = _ffi.SgPairFile()
    _check(_ffi.load().sg_read_pairs(path.encode(), 0 if fmt == "tsv" else 1, C.byref(out)))
    return PairFile(out)


def write_results(path: Optional[str], pairs: PairFile, res: "Results", json: bool = False) -> None:
    """write_batch_tsv (batch.cpp:106-113) or the CLI's JSON (main.cpp:77-88)."""
    _check(_ffi.load().sg_write_results(path.encode() if path else None, C.byref(pairs._f),
                                        C.byref(res._res), int(bool(json))))


def synth_packed(cfg_id: int, first: int = 0, count: int = -1) -> PackedBatch:
    """BASELINE config `cfg_id` pairs [first, first+count), 2-bit packed (csrc/synth.h)."""
    out = _ffi.SgPackedPairs()
    _check(_ffi.load().sg_synth_packed(cfg_id, first, count, C.byref(out)))
    return PackedBatch(out)


def synth_codes(cfg_id: int, first: int = 0, count: int = -1) -> CodesBatch:
    out = _ffi.SgPairs()
    _check(_ffi.load().sg_synth_codes(cfg_id, first, count, C.byref(out)))
    n = out.n_pairs
    arr = lambda p, t, k: np.ctypeslib.as_array(C.cast(p, C.POINTER(t)), (max(k, 1),))[:k]
    tl = arr(out.text_len, C.c_int64, n)
    pl = arr(out.pat_len, C.c_int64, n)
    text = arr(out.text, C.c_uint8, int(tl.sum()))
    pattern = arr(out.pattern, C.c_uint8, int(pl.sum()))
    return CodesBatch(text, arr(out.text_off, C.c_int64, n), tl, pattern,
                      arr(out.pat_off, C.c_int64, n), pl, owner=out)


def last_transfer_bytes():
    L = _ffi.load()
    return int(L.sg_last_transfer_bytes(0)), int(L.sg_last_transfer_bytes(1))


@contextlib.contextmanager
def options(kernel: Optional[str] = None, stream_upload: Optional[bool] = None,
            longest_first: Optional[bool] = None, diagnostics: Optional[int] = None,
            exact_budget: Optional[int] = None):
    """Process-wide execution options (sg_set_options) for the duration of a block:
    which K1 runs ("auto", "full", "mixed", "wide"), the streamed upload, the
    longest-first order, diagnostics bits and K7's memory budget. They pick among
    equivalent device paths for cross-checks and measurements; none changes a result."""
    L = _ffi.load()
    old = _ffi.SgOptions()
    L.sg_get_options(C.byref(old))
    new = _ffi.SgOptions()
    C.memmove(C.byref(new), C.byref(old), C.sizeof(old))
    if kernel is not None:
        new.kernel = _ffi.SG_KERNEL[kernel]
    if stream_upload is not None:
        new.stream_upload = int(bool(stream_upload))
    if longest_first is not None:
        new.longest_first = int(bool(longest_first))
    if diagnostics is not None:
        new.diagnostics = int(diagnostics)
    if exact_budget is not None:
        new.exact_budget = int(exact_budget)
    _check(L.sg_set_options(C.byref(new)))
    try:
        yield
    finally:
        L.sg_set_options(C.byref(old))


class Session:
    """Device-resident batch on one GPU: inputs uploaded once, kernels re-run."""

    def __init__(self, config: AlignerConfig, batch: PackedBatch, device: int = 0):
        self._h = C.c_void_p()
        self.batch = batch
        _check(_ffi.load().sg_session_create(C.byref(config._c()), C.byref(batch.c), device,
                                             C.byref(self._h)))

    def run(self):
        """Runs K1-K3 once; returns (device_ms of K1-K3, K1 ms) from CUDA events."""
        ms, k1 = C.c_float(), C.c_float()
        _check(_ffi.load().sg_session_run(self._h, C.byref(ms), C.byref(k1)))
        return ms.value, k1.value

    def fetch(self) -> Results:
        res = _ffi.SgResults()
        _check(_ffi.load().sg_session_fetch(self._h, C.byref(res)))
        return Results(res)

    def info(self):
        lanes, sms, limbs = C.c_int64(), C.c_int32(), C.c_int32()
        _ffi.load().sg_session_info(self._h, C.byref(lanes), C.byref(sms), C.byref(limbs))
        kernel = ("full", "mixed", "wide")[_ffi.load().sg_session_kernel(self._h)]
        return {"lanes": lanes.value, "sms": sms.value, "limbs": limbs.value, "kernel": kernel}

    def phase_cycles(self):
        """Per-phase cycle counters of the last run under options(diagnostics=2)."""
        buf = (C.c_uint64 * 25)()
        if _ffi.load().sg_session_phase_cycles(self._h, buf) != 0:
            return None
        return list(buf)

    def warp_times(self, cap: int = 8192):
        """(start, exit, smid) per warp of the last run under options(diagnostics=1)."""
        buf = (C.c_uint64 * (3 * cap))()
        n = _ffi.load().sg_session_warp_times(self._h, buf, cap)
        if n < 0:
            return None
        return [tuple(buf[3 * k:3 * k + 3]) for k in range(n)]

    def close(self):
        if self._h:
            _ffi.load().sg_session_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------- reference-shaped API

def _outcome(res: Results, k: int) -> PairOutcome:
    return PairOutcome(bool(res.found[k]), int(res.distance[k]), res.cigar(k),
                       int(res.windows[k]), res.pair_counters(k))


def align(text, pattern, config: Optional[AlignerConfig] = None) -> AlignmentResult:
    """align (proj/src/aligner.cpp:28-85) for one pair; text/pattern are codes or strings."""
    config = config or AlignerConfig()
    if config.mode != "windowed":
        if config.mode == "single":
            raise ConfigError("align() requires windowed mode")
        raise ConfigError(f"unknown mode '{config.mode}'")
    config.validate()
    t, p = encode_sequence(text), encode_sequence(pattern)
    if not t or not p:
        raise InputError("align: empty input sequence")
    res = align_codes(config, CodesBatch.from_lists([t], [p]))
    o = _outcome(res, 0)
    return AlignmentResult(o.distance, o.cigar, o.windows, o.counters)


def run_batch(pairs: Sequence[SeqPairRecord], config: Optional[AlignerConfig] = None,
              threads: int = 1, devices=None) -> BatchResult:
    """run_batch (proj/src/batch.cpp:13-104) on the GPU(s); `threads` is accepted for
    signature parity (host threads are sized by the runtime)."""
    config = config or AlignerConfig()
    config.validate()
    if threads < 1:
        raise ConfigError("thread count must be at least 1")
    ids = [p.id for p in pairs]
    for p in pairs:
        if not p.text or not p.pattern:
            raise InputError(f"pair '{p.id}': empty sequence")
    batch = CodesBatch.from_lists([encode_sequence(p.text) for p in pairs],
                                  [encode_sequence(p.pattern) for p in pairs])
    res = align_codes(config, batch, devices, ids)
    out = BatchResult(outcomes=[_outcome(res, k) for k in range(res.n)], total=res.total,
                      align_seconds=res.align_seconds, device_ms=res.device_ms,
                      kernel_ms=res.kernel_ms, gpu_launches=int(res.gpu_launches))
    out.pairs_per_second = len(pairs) / out.align_seconds if out.align_seconds > 0 else 0.0
    return out


def write_batch_tsv(f, pairs: Sequence[SeqPairRecord], result: BatchResult) -> None:
    """write_batch_tsv (proj/src/batch.cpp:106-113)."""
    for p, o in zip(pairs, result.outcomes):
        f.write(f"{p.id}\t{o.distance}\t{cigar_to_string(o.cigar) if o.found else '*'}\n")


# ---------------------------------------------------------------- accuracy sweep
# run_sweep (proj/src/sweep.cpp:40-107) with the GPU exact
# oracle (K7, sg_global_align) in place of the quadratic CPU global_align.

@dataclass
class ScoringParams:
    """oracle::ScoringParams (proj/include/scrooge/oracle.hpp:14-19)."""
    match_bonus: int = 2
    mismatch_penalty: int = 4
    gap_open: int = 4
    gap_extend: int = 2

    def _c(self) -> _ffi.SgScoring:
        return _ffi.SgScoring(self.match_bonus, self.mismatch_penalty, self.gap_open,
                              self.gap_extend)


def score_cigar(cigar: Iterable, params: Optional[ScoringParams] = None) -> int:
    """oracle::score_cigar (proj/src/oracle.cpp:91-115): affine gap score of a CIGAR."""
    params = params or ScoringParams()
    score, prev = 0, ""
    for op, n in cigar:
        if op not in "=XID":
            raise InputError(f"score_cigar: unknown op '{op}'")
        if n <= 0:
            raise InputError("score_cigar: non-positive run length")
        if op == "=":
            score += params.match_bonus * n
        elif op == "X":
            score -= params.mismatch_penalty * n
        elif op == prev:
            score -= params.gap_extend * n
        else:
            score -= params.gap_open + params.gap_extend * n
        prev = op
    return score


def worst_quantile(scores: Sequence[int], p: float) -> int:
    """worst_quantile (proj/src/sweep.cpp:11-19), through the library."""
    arr = (C.c_int64 * len(scores))(*scores)
    out = C.c_int64()
    _check(_ffi.load().sg_worst_quantile(arr, len(scores), p, C.byref(out)))
    return out.value


def global_align_packed(batch, device: int = 0) -> Results:
    """oracle::global_align (proj/src/oracle.cpp:39-89) for every pair, on the GPU (K7)."""
    res = _ffi.SgResults()
    _check(_ffi.load().sg_global_align(C.byref(batch.c), device, C.byref(res)))
    return Results(res)


@dataclass
class GlobalAlignment:
    distance: int
    cigar: Cigar


def global_align(text, pattern, device: int = 0) -> GlobalAlignment:
    """oracle::global_align for one pair (codes or strings), on the GPU."""
    b = pack(CodesBatch.from_lists([encode_sequence(text)], [encode_sequence(pattern)]))
    r = global_align_packed(b, device)
    return GlobalAlignment(int(r.distance[0]), r.cigar(0))


@dataclass
class SweepRow:
    """SweepRow (proj/include/scrooge/sweep.hpp:42-53)."""
    W: int
    O: int
    sene: bool
    dent: bool
    et: bool
    q500: int
    q100: int
    q010: int
    q001: int
    frac_optimal: float
    mean_rows_frac: float
    stored_bits_ratio: float
    pairs_per_s: float
    oracle_q500: int
    oracle_q100: int
    oracle_q010: int
    oracle_q001: int


_COMBO_FLAGS = {"sene": 1, "dent": 2, "et": 4}


def _combo_bits(c) -> int:
    if isinstance(c, int):
        return c
    if isinstance(c, str):
        bits = 0
        if c != "none":
            for f in c.split("+"):
                if f not in _COMBO_FLAGS:
                    raise InputError(f"unknown improvement '{f}' (expected sene, dent, et, none or all)")
                bits |= _COMBO_FLAGS[f]
        return bits
    sene, dent, et = c
    return int(bool(sene)) | (int(bool(dent)) << 1) | (int(bool(et)) << 2)


def _rows_c(rows):
    arr = (_ffi.SgSweepRow * len(rows))()
    for k, r in enumerate(rows):
        arr[k] = _ffi.SgSweepRow(r.W, r.O, int(r.sene), int(r.dent), int(r.et), r.q500, r.q100,
                                 r.q010, r.q001, r.frac_optimal, r.mean_rows_frac,
                                 r.stored_bits_ratio, r.pairs_per_s, r.oracle_q500,
                                 r.oracle_q100, r.oracle_q010, r.oracle_q001)
    return arr


def run_sweep(pairs, W_list: Sequence[int] = (32, 64), o_rule="half+1",
              combos=("none", "sene+dent+et"), scoring: Optional[ScoringParams] = None,
              devices=None, measure_time: bool = True) -> List[SweepRow]:
    """run_sweep (proj/src/sweep.cpp:40-107) on the GPU. pairs: SeqPairRecords or a
    packed batch; o_rule "half+1" or "fixed:<n>" (or an int); combos: "none",
    "sene+dent+et", ..., "all", or (sene, dent, et) tuples."""
    if not isinstance(pairs, (PackedBatch, _PackedView)):
        pairs = list(pairs)
        n = len(pairs)
        batch = pack(CodesBatch.from_lists([encode_sequence(p.text) for p in pairs],
                                           [encode_sequence(p.pattern) for p in pairs])) if n else None
    else:
        batch = pairs
        n = batch.c.n_pairs
    bits = []
    for c in combos:
        if c == "all":
            bits.extend(range(8))
        else:
            bits.append(_combo_bits(c))
    if isinstance(o_rule, int):
        o_fixed = o_rule
    elif o_rule == "half+1":
        o_fixed = -1
    elif isinstance(o_rule, str) and o_rule.startswith("fixed:"):
        o_fixed = int(o_rule[6:])
    else:
        raise InputError(f"unknown O rule '{o_rule}'")
    Ws = (C.c_int32 * len(W_list))(*W_list)
    cs = (C.c_uint8 * max(len(bits), 1))(*bits)
    opt = _ffi.SgSweepOptions(Ws, len(W_list), o_fixed, cs, len(bits),
                              (scoring or ScoringParams())._c(), int(measure_time))
    rows = (_ffi.SgSweepRow * max(len(W_list) * len(bits), 1))()
    darr, nd = _devices(devices)
    _check(_ffi.load().sg_sweep(C.byref(opt), C.byref(batch.c) if n else None, darr, nd, rows))
    out = []
    for k in range(len(W_list) * len(bits)):
        r = rows[k]
        out.append(SweepRow(r.W, r.O, bool(r.sene), bool(r.dent), bool(r.et), r.q500, r.q100,
                            r.q010, r.q001, r.frac_optimal, r.mean_rows_frac,
                            r.stored_bits_ratio, r.pairs_per_s, r.oracle_q500, r.oracle_q100,
                            r.oracle_q010, r.oracle_q001))
    return out


def _sweep_format(rows: Sequence[SweepRow], json: bool) -> str:
    arr = _rows_c(rows)
    L = _ffi.load()
    n = L.sg_sweep_format(arr, len(rows), int(json), None, 0)
    buf = C.create_string_buffer(n + 1)
    L.sg_sweep_format(arr, len(rows), int(json), buf, n + 1)
    return buf.value.decode()


def sweep_csv(rows: Sequence[SweepRow]) -> str:
    """sweep_csv (proj/src/sweep.cpp:110-127)."""
    return _sweep_format(rows, False)


def sweep_json(rows: Sequence[SweepRow]) -> str:
    """The CLI's sweep JSON (proj/tools/main.cpp:90-111, dump(2))."""
    return _sweep_format(rows, True)
