/*
 * scrooge_b200 — C ABI of the B200-native windowed GenASM aligner.
 *
 * This is the drop-in boundary for the reference's aligner path
 * (/root/reference/proj/include/scrooge/). Plain C types only; no exceptions
 * cross it. The C++ shim (include/scrooge_b200.hpp) and the Python package
 * (paper_2208_09985_b200) re-raise the reference's exception types from the
 * status codes below.
 *
 *   reference                                       replaced by
 *   ------------------------------------------------------------------------
 *   AlignerConfig            aligner.hpp:12-31      sg_config
 *   AlignerConfig::validate  aligner.cpp:8-18       sg_validate_config
 *   align()                  aligner.hpp:45,        sg_align_batch (n_pairs = 1)
 *                            aligner.cpp:28-85
 *   run_batch()              batch.hpp:33-34,       sg_align_batch / sg_align_packed
 *                            batch.cpp:13-104
 *   PairOutcome/BatchResult  batch.hpp:14-27        sg_results
 *   InstrumentationCounters  dp.hpp:46-66           sg_results.counters
 *   cigar_to_string          cigar.cpp:18-25        sg_cigar_string
 *   write_batch_tsv          batch.cpp:106-113      sg_results + sg_cigar_string
 *   encode_sequence          sequence.hpp:19-37     codes in sg_pairs (1 B/base)
 *   InputError / ConfigError / InternalError        SG_INPUT / SG_CONFIG / SG_INTERNAL
 *                            errors.hpp:10-34
 *
 * Semantics: identical edit distance and CIGAR to the reference for every
 * pair at the same (W, O, sene, dent, early_termination). The switches change
 * work and footprint in the reference, not results (proj/tests/acceptance.cpp:
 * 93-126). On the GPU early_termination changes the work the same way: with it
 * a window stops at the first row d with D(0, 0) <= d (dp.cpp:177, in chunks of
 * 4 rows); without it every kernel computes all K + 1 rows of every window
 * (dp.cpp:225; such batches run the full-frame K1 or K6). sene / dent select the
 * reference's storage policy, whose counters are reported; the device itself
 * always keeps 2-bit traceback events for the columns the traceback can reach
 * (DENT's region), never the reference's table.
 */
#ifndef SCROOGE_B200_H
#define SCROOGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 1

/* Status codes (proj/tools/main.cpp:287-299 maps the same classes to exit codes). */
enum {
    SG_OK = 0,
    SG_INPUT = 1,    /* scrooge::InputError */
    SG_CONFIG = 2,   /* scrooge::ConfigError */
    SG_INTERNAL = 3, /* scrooge::InternalError (incl. OutOfStoredRegionError) */
    SG_CUDA = 4      /* device / driver failure (no reference equivalent) */
};

/* AlignerConfig, proj/include/scrooge/aligner.hpp:12-31. Defaults W=64, O=33,
 * all switches on (sg_config_default). single_window selects
 * Mode::SingleWindow (align_single_window, aligner.cpp:87-112) with edit budget
 * k_single; sequences of up to 1024 characters (K1 up to 128, K6 above). */
typedef struct sg_config {
    int32_t W;
    int32_t O;
    uint8_t sene;
    uint8_t dent;
    uint8_t early_termination;
    uint8_t single_window;
    int32_t k_single;
} sg_config;

/* Pairs as 1-byte base codes (proj/include/scrooge/sequence.hpp:13-16:
 * 0..3 = A,C,G,T; anything else = non-ACGT, matches nothing).
 * Sequence k of the batch is text[text_off[k] .. text_off[k] + text_len[k]). */
typedef struct sg_pairs {
    int64_t n_pairs;
    const uint8_t* text;
    const int64_t* text_off;
    const int64_t* text_len;
    const uint8_t* pattern;
    const int64_t* pat_off;
    const int64_t* pat_len;
} sg_pairs;

/* Pairs already 2-bit packed (BASELINE cfg2's input form): 16 bases per word,
 * base k at bits 2(k%16)..2(k%16)+1 of word k/16 (A=0 C=1 G=2 T=3). Offsets
 * are in bases. nmask (optional, NULL = pure ACGT) holds 1 bit per base at the
 * same offsets (bit k%32 of word k/32); a set bit marks a non-ACGT base. */
typedef struct sg_packed_pairs {
    int64_t n_pairs;
    const uint32_t* seq;
    int64_t seq_words;
    const uint32_t* nmask;
    const int64_t* text_off;
    const int64_t* text_len;
    const int64_t* pat_off;
    const int64_t* pat_len;
} sg_packed_pairs;

/* Run encoding of CIGARs: one byte per run piece, (op << 6) | (len - 1),
 * op 0 '=', 1 'X', 2 'I', 3 'D', len 1..64. Consecutive bytes with the same
 * op continue one run (cigar_append merges, proj/src/cigar.cpp:9-16, so two
 * real runs never share an op). */
enum { SG_OP_MATCH = 0, SG_OP_SUB = 1, SG_OP_INS = 2, SG_OP_DEL = 3 };

/* Counter slots per pair, InstrumentationCounters order (dp.hpp:46-66). */
enum {
    SG_CNT_STORED_BITS = 0,
    SG_CNT_TABLE_WRITES,
    SG_CNT_TABLE_READS,
    SG_CNT_ROWS_COMPUTED,
    SG_CNT_CELLS_COMPUTED,
    SG_CNT_ROWS_POSSIBLE,
    SG_CNT_BASELINE_EQUIV_BITS,
    SG_CNT_COUNT
};

/* PairOutcome / BatchResult, proj/include/scrooge/batch.hpp:14-27, in input order. */
typedef struct sg_results {
    int64_t n_pairs;
    int64_t* distance;     /* [n] */
    int32_t* windows;      /* [n] */
    uint8_t* found;        /* [n] (always 1 in windowed mode) */
    int64_t* cigar_off;    /* [n+1] byte offsets into runs */
    uint8_t* runs;         /* run bytes, see SG_OP_* */
    uint64_t* counters;    /* [n][SG_CNT_COUNT] */
    uint64_t total[SG_CNT_COUNT]; /* BatchResult::total */
    double align_seconds;  /* host wall time of the whole call (H2D + kernels + D2H) */
    double device_ms;      /* device time of the kernels (CUDA events, max over devices) */
    double kernel_ms;      /* device time of K1 alone (max over devices) */
    int64_t gpu_launches;  /* kernels launched by this call */
    void* _owner;          /* internal */
} sg_results;

/* Library info. */
int sg_abi_version(void);
int sg_device_count(void);
const char* sg_last_error(void); /* message of the last failing call on this thread */

void sg_config_default(sg_config* cfg);
/* AlignerConfig::validate (aligner.cpp:8-18) + GPU-path limits. */
int sg_validate_config(const sg_config* cfg);

/* run_batch over 1-byte codes: validates, packs (host threads), shards the
 * pairs over `devices` (NULL = device 0; n_devices >= 1), runs K1-K3, copies
 * results back. Blocking. On SG_INPUT / SG_INTERNAL the message names the
 * first failing pair by index ("pair '<index>': ..."), as batch.cpp:69-77. */
int sg_align_batch(const sg_config* cfg, const sg_pairs* pairs, const int* devices,
                   int n_devices, sg_results* out);
/* Same over 2-bit packed input (no host packing). */
int sg_align_packed(const sg_config* cfg, const sg_packed_pairs* pairs, const int* devices,
                    int n_devices, sg_results* out);
void sg_results_free(sg_results* res);

/* cigar_to_string of pair k: writes "<len><op>..." + NUL into buf when it fits;
 * returns the string length (excl. NUL), or -1 on a bad index. */
int64_t sg_cigar_string(const sg_results* res, int64_t k, char* buf, int64_t cap);
/* Decoded runs of pair k into ops[] ('=','X','I','D') / lens[]; returns the
 * run count (may exceed cap: then only cap runs are written). */
int64_t sg_cigar_runs(const sg_results* res, int64_t k, char* ops, int64_t* lens, int64_t cap);

/* 2-bit packing (K4) of 1-byte codes with host threads. The packed buffers are
 * owned by `out` and released with sg_packed_free. Each sequence starts on a
 * word boundary. */
int sg_pack(const sg_pairs* in, sg_packed_pairs* out);
void sg_packed_free(sg_packed_pairs* p);

/* K5, the device split of a batch, on the host alone: pair k goes
 * to device slot shard[k] (0 .. n_devices-1) at position pos[k] of that device's
 * batch. *gathered = 0 when the shards are contiguous ranges of input order
 * (pairs of near-equal estimated cost), 1 when the pairs were sorted into cost
 * buckets and dealt longest-first to the least-loaded device (cfg5's mix).
 * sg_align_batch / sg_align_packed use exactly this split for n_devices > 1. */
int sg_plan_shards(const sg_packed_pairs* pairs, int n_devices, int32_t* shard, int64_t* pos,
                   int* gathered);

/* Bytes copied host->device (direction 0) / device->host (1) by the last
 * sg_align_batch / sg_align_packed call on this thread. */
int64_t sg_last_transfer_bytes(int direction);

/* Process-wide execution options. They select among equivalent device paths for
 * cross-checks, A/B measurements and diagnostics; no option changes a result.
 * Defaults (sg_options_default) are what the library picks on its own. Set them
 * between calls, not while a call is running. */
enum {
    SG_KERNEL_AUTO = 0,   /* the host's choice per shard */
    SG_KERNEL_FULL = 1,   /* full-frame K1 (one pair per lane) */
    SG_KERNEL_MIXED = 2,  /* mixed band / cooperative K1 where the window shape allows */
    SG_KERNEL_WIDE = 3    /* K6 (one pair per warp) for every batch */
};
enum {
    SG_DIAG_WARP_TIMES = 1,   /* per-warp start/exit timeline of sessions' K1 */
    SG_DIAG_PHASE_CYCLES = 2, /* per-phase SM cycles of sessions' K1 */
    SG_DIAG_HOST_TRACE = 4,   /* host pipeline timestamps on stderr */
    SG_DIAG_NO_PIPELINE = 8   /* one-shot calls launch the mixed kernel's tail kernels after it,
                                 not beside it: A/B and cross-checks */
};
typedef struct sg_options {
    int32_t kernel;         /* SG_KERNEL_* */
    int32_t stream_upload;  /* 1: one-shot calls overlap the sequence H2D with K1 */
    int32_t longest_first;  /* 1: pairs of different lengths start longest first */
    int32_t diagnostics;    /* SG_DIAG_* bits */
    int64_t exact_budget;   /* K7 delta-store bytes per batch; 0 = half the free memory */
} sg_options;
void sg_options_default(sg_options* o);
int sg_set_options(const sg_options* o); /* SG_CONFIG for an unknown kernel */
void sg_get_options(sg_options* o);

/* Device-resident sessions (inputs already in HBM when timing starts). */
typedef struct sg_session sg_session;
int sg_session_create(const sg_config* cfg, const sg_packed_pairs* pairs, int device,
                      sg_session** out);
/* Runs K1-K3 once on the session's stream; returns device ms (CUDA events). */
int sg_session_run(sg_session* s, float* device_ms, float* k1_ms);
int sg_session_fetch(sg_session* s, sg_results* out);
/* Per-session facts for the roofline: resident lanes, SMs, K1 launches. */
int sg_session_info(const sg_session* s, int64_t* lanes, int32_t* sms, int32_t* limbs);
/* Which K1 the session runs: 0 the full-frame kernel, 1 the mixed
 * band / cooperative kernel, 2 the wide-window kernel K6. Diagnostics; no reference
 * counterpart. */
int sg_session_kernel(const sg_session* s);
void sg_session_destroy(sg_session* s);
/* Diagnostics of the session's last run with SG_DIAG_PHASE_CYCLES / SG_DIAG_WARP_TIMES
 * set: 25 per-phase counters (setup, DC, TB, ... cycles summed over warps), or
 * per-warp (start, exit, smid) triples (returns the warp count, <= cap). -1 when
 * the run did not collect them. */
int sg_session_phase_cycles(sg_session* s, uint64_t* out25);
int sg_session_warp_times(sg_session* s, uint64_t* out, int cap);

/* Measured integer-ALU issue rate of `device` (LOP3 lane-ops per clock per SM,
 * the clock the microbenchmark ran at, and lane-ops/s) — the roofline
 * denominator for K1. */
int sg_alu_peak(int device, double* ops_per_clk_per_sm, double* sm_mhz, double* ops_per_s);

/* Seeded synthetic pairs of the BASELINE configs (paper_2208_09985_b200/csrc/
 * synth.h), generated straight into packed form with host threads. */
int sg_synth_packed(int cfg_id, int64_t first, int64_t count, sg_packed_pairs* out);
/* Same pairs as 1-byte codes (buffers owned by out, free with sg_pairs_free). */
int sg_synth_codes(int cfg_id, int64_t first, int64_t count, sg_pairs* out);
void sg_pairs_free(sg_pairs* p);

/* ---- pair files and result output (the CLI's data path) ----------------
 * sg_read_pairs reads the reference's pair formats straight into packed form:
 *   SG_FORMAT_TSV        `id<TAB>text<TAB>pattern` per line (read_pairs_tsv,
 *                        proj/src/io.cpp:66-94);
 *   SG_FORMAT_FASTA_PAIR "<text.fa>,<pattern.fa>", records paired in order
 *                        (read_pairs_fasta, io.cpp:96-112; read_pairs io.cpp:114-121).
 * Sequences are upper-cased; CR line ends and empty lines are skipped; ids
 * must be unique. Errors are SG_INPUT with the reference's messages.
 * sg_write_results writes `id<TAB>distance<TAB>cigar` lines, "*" for a pair
 * that was not found (write_batch_tsv, proj/src/batch.cpp:106-113), or with
 * json != 0 the CLI's JSON array (proj/tools/main.cpp:77-88). path NULL or
 * "-" writes to stdout. */
enum { SG_FORMAT_TSV = 0, SG_FORMAT_FASTA_PAIR = 1 };
typedef struct sg_pair_file {
    int64_t n_pairs;
    const char* const* ids;  /* [n_pairs] NUL-terminated */
    sg_packed_pairs packed;  /* owned; pass to sg_align_packed */
    void* _owner;
} sg_pair_file;
int sg_read_pairs(const char* input, int format, sg_pair_file* out);
void sg_pair_file_free(sg_pair_file* f);
int sg_write_results(const char* path, const sg_pair_file* pairs, const sg_results* res, int json);

/* ---- exact global alignment and the accuracy sweep ------
 * sg_global_align: the optimal unit-cost global alignment of every pair with
 * the reference oracle's tie-breaking (oracle::global_align,
 * proj/src/oracle.cpp:39-89), on `device` (K7). Results as sg_align_packed
 * (windows = 1, found = 1, counters 0). The reference's guards apply: a
 * sequence over 10^5 bases, or (n+1)(m+1) > 2^30, is SG_INPUT with its
 * message (oracle.cpp:43-46). */
int sg_global_align(const sg_packed_pairs* pairs, int device, sg_results* out);

/* oracle::ScoringParams (proj/include/scrooge/oracle.hpp:14-19) and
 * oracle::score_cigar (oracle.cpp:91-115) of pair k's CIGAR. */
typedef struct sg_scoring {
    int32_t match_bonus, mismatch_penalty, gap_open, gap_extend;
} sg_scoring;
void sg_scoring_default(sg_scoring* s); /* 2, 4, 4, 2 */
int64_t sg_score_cigar(const sg_results* res, int64_t k, const sg_scoring* s);
/* worst_quantile (proj/src/sweep.cpp:11-19): the ceil(p n)-th lowest score. */
int sg_worst_quantile(const int64_t* scores, int64_t n, double p, int64_t* out);

/* run_sweep (proj/src/sweep.cpp:40-107) with the GPU for both the aligner
 * (sg_align_packed per W and combo) and the exact oracle (sg_global_align).
 * SweepOptions (proj/include/scrooge/sweep.hpp:12-40): */
typedef struct sg_sweep_options {
    const int32_t* W_list;
    int32_t n_W;
    int32_t o_fixed;        /* OverlapRule: -1 = W/2 + 1 (HalfPlusOne), else this fixed O */
    const uint8_t* combos;  /* ImprovementCombo per entry: bit 0 sene, bit 1 dent, bit 2 et */
    int32_t n_combos;
    sg_scoring scoring;
    int32_t measure_time;   /* 0: pairs_per_s = 0, for byte-stable reports */
} sg_sweep_options;
/* SweepRow (sweep.hpp:42-53). */
typedef struct sg_sweep_row {
    int32_t W, O;
    uint8_t sene, dent, et;
    int64_t q500, q100, q010, q001;
    double frac_optimal, mean_rows_frac, stored_bits_ratio, pairs_per_s;
    int64_t oracle_q500, oracle_q100, oracle_q010, oracle_q001;
} sg_sweep_row;
/* rows: n_W * n_combos entries, W-major (the reference's order). Errors as
 * the reference: SG_INPUT for an empty dataset / W list / combo list or an
 * oversized pair, SG_CONFIG for an invalid (W, O). */
int sg_sweep(const sg_sweep_options* opt, const sg_packed_pairs* pairs, const int* devices,
             int n_devices, sg_sweep_row* rows);
/* sweep_csv (sweep.cpp:110-127), or with json != 0 the CLI's JSON
 * (proj/tools/main.cpp:90-111, dump(2)). Returns the length; writes the text
 * and a NUL into buf when it fits. */
int64_t sg_sweep_format(const sg_sweep_row* rows, int64_t n_rows, int json, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* SCROOGE_B200_H */
