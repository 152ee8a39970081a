"""paper_2208_09985_b200 — B200-native windowed GenASM aligner (Scrooge, arXiv 2208.09985).

GenASM-DC + GenASM-TB + the window loop as hand-written sm_100a CUDA kernels
behind a C ABI (include/scrooge_b200.h); this package mirrors the reference's
C++ aligner API (proj/include/scrooge/) on top of it. See DESIGN.md.
"""
from .aligner import (  # noqa: F401
    AlignerConfig, AlignmentResult, BatchResult, CodesBatch, ConfigError, CudaError,
    InputError, InstrumentationCounters, InternalError, OutOfStoredRegionError, PackedBatch,
    PairOutcome, Results, SeqPairRecord, Session, align, align_codes, align_packed,
    cigar_from_string, cigar_to_string, decode_sequence, encode_sequence, last_transfer_bytes,
    pack, run_batch, synth_codes, synth_packed, write_batch_tsv, PairFile, read_pairs,
    write_results, ScoringParams, score_cigar, worst_quantile, global_align,
    global_align_packed, GlobalAlignment, SweepRow, run_sweep, sweep_csv, sweep_json, options,
)
from .build import LIB as LIBRARY_PATH  # noqa: F401
