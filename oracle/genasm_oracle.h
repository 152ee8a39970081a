/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's windowed GenASM aligner
 * (/root/reference/proj/src/{aligner,dp,traceback,cigar}.cpp). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker or the CPU baseline. The product path
 * (paper_2208_09985_b200) never links or calls it.
 *
 * Parity pin: tests/test_oracle_pin.py checks this restatement against golden
 * vectors produced by the reference itself (oracle/_ref/ref_tool, built from
 * the reference sources by oracle/Makefile; fixtures in tests/golden/).
 */
#ifndef GENASM_ORACLE_H
#define GENASM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/include/scrooge/aligner.hpp:12-31 */
typedef struct orc_config {
    int32_t W, O;
    uint8_t sene, dent, et;
    uint8_t single_window; /* Mode::SingleWindow */
    int32_t k_single;
} orc_config;

/* proj/include/scrooge/dp.hpp:46-66 */
typedef struct orc_counters {
    uint64_t stored_bits, table_writes, table_reads, rows_computed, cells_computed,
        rows_possible, baseline_equiv_bits;
} orc_counters;

typedef struct orc_result {
    int32_t found;    /* 0 only in single-window mode past k */
    int64_t distance; /* -1 when !found */
    int32_t windows;
    int64_t n_runs;
    char* ops;        /* run ops '=', 'X', 'I', 'D' (malloc'ed) */
    int64_t* lens;    /* run lengths (malloc'ed) */
    orc_counters counters;
} orc_result;

enum { ORC_OK = 0, ORC_INPUT = 1, ORC_CONFIG = 2, ORC_INTERNAL = 3 };

/* align() (proj/src/aligner.cpp:28-85) or align_single_window() (:87-112)
 * depending on cfg->single_window. Codes 0..3 = ACGT, 4 = other. */
int orc_align(const orc_config* cfg, const uint8_t* text, int64_t n, const uint8_t* pattern,
              int64_t m, orc_result* out, char* err, size_t errlen);
void orc_result_free(orc_result* r);

/* cigar_to_string (proj/src/cigar.cpp:18-25); returns bytes written (excl. NUL),
 * or the required size when buf is too small. */
int64_t orc_cigar_string(const orc_result* r, char* buf, int64_t cap);

/* validate_replay (proj/src/cigar.cpp:70-107) over the compact run bytes of
 * the GPU path ((op << 6) | (len - 1), op 0 '=', 1 'X', 2 'I', 3 'D';
 * same-op bytes continue a run). Returns the edit count (X + I + D), or -1 if
 * the CIGAR does not transform text into pattern. */
int64_t orc_replay_runs(const uint8_t* text, int64_t n, const uint8_t* pattern, int64_t m,
                        const uint8_t* runs, int64_t nbytes);
/* Same check for many pairs at once (threads); returns the number of pairs
 * that fail or whose edit count differs from distance[k]. */
int64_t orc_replay_batch(int64_t n_pairs, const uint8_t* text, const int64_t* text_off,
                         const int64_t* text_len, const uint8_t* pattern, const int64_t* pat_off,
                         const int64_t* pat_len, const uint8_t* runs, const int64_t* cigar_off,
                         const int64_t* distance, int threads);

/* Per-window statistics hook: d_opt and window geometry of every window of
 * the last orc_align call on this thread (for ALG_OPS/design studies). */
int64_t orc_last_window_count(void);
void orc_last_window_stats(int32_t* d_opt, int32_t* n_w, int32_t* m_w, int64_t cap);

/* oracle::global_align (proj/src/oracle.cpp:39-89): optimal unit-cost global
 * alignment, forward DP with the choice order diagonal > delete > insert
 * (strict improvements only), traceback from (n, m). Fills distance, runs
 * (windows = 1, found = 1). ORC_INPUT for the reference's size guards. */
int orc_global_align(const uint8_t* text, int64_t n, const uint8_t* pattern, int64_t m,
                     orc_result* out, char* err, size_t errlen);
/* oracle::score_cigar (oracle.cpp:91-115) of a result's runs. */
int64_t orc_score_cigar(const orc_result* r, int match_bonus, int mismatch_penalty, int gap_open,
                        int gap_extend);
/* worst_quantile (proj/src/sweep.cpp:11-19); scores are sorted in place. */
int64_t orc_worst_quantile(int64_t* scores, int64_t n, double p);

/* Per-block digests of a batch's results, as `ref_tool digest` computes them from
 * the reference's BatchResult (oracle/ref_tool.cpp:digest_line): per pair the line
 * "distance\tfnv(cigar_to_string)\truns\twindows\t<7 counters>\n" (the CIGAR of a
 * not-found pair is "*"), and per block of `block` pairs fnv1a64 over its lines.
 * Inputs are the GPU path's sg_results arrays (run bytes as orc_replay_runs).
 * Writes ceil(n/block) digests; returns fnv1a64 over their 16-hex-digit forms. */
uint64_t orc_digest_blocks(int64_t n_pairs, const int64_t* distance, const int32_t* windows,
                           const uint8_t* found, const int64_t* cigar_off, const uint8_t* runs,
                           const uint64_t* counters, int64_t block, uint64_t* digests,
                           int threads);

#ifdef __cplusplus
}
#endif

#endif
