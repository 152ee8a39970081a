// K1 `window_align`: the fused GenASM-DC + GenASM-TB + window loop (sm_100a).
//
// Replaces compute_dc (proj/src/dp.cpp:104-231), traceback
// (proj/src/traceback.cpp:56-113) and the window loop of align
// (proj/src/aligner.cpp:28-85). See DESIGN.md §3 for the derivation; summary:
//
//  * One thread owns one pair (SIMT across pairs). A persistent grid pulls
//    pairs from an atomic queue (optionally in a caller-given order).
//  * Bit vectors are 32L-bit registers ("limbs"), logical position q = pL + r
//    lives in limb r, machine bit 31-p. The pattern is right-aligned
//    (bit j at q = j + 32L - m_w), so the end-of-pattern boundary bit
//    (proj/include/scrooge/dp.hpp:145-154) always enters at the LSB of limb
//    L-1 and a DP shift costs ONE integer multiply-add (x*2 + b, FMA pipe):
//    the other limbs are renamed, not moved.
//  * DC sweeps columns i = n-1..0 and keeps R rows of the column in registers
//    (rows d0..d0+R-1, a "chunk"). Early termination is per lane at chunk
//    granularity: a lane whose window is not solved continues with the next
//    chunk (the last row of each column is parked in a global scratch row)
//    while its warp-mates already trace back or start their next window.
//  * SENE/DENT: nothing of R is retained. For the DENT region (columns
//    < C, C >= W-O) each cell keeps a 2-bit traceback code accumulated
//    during DC from the SENE regeneration rule evaluated at the cell's own
//    row (traceback.cpp:35-54): Match <=> t_i == p_j; Sub <=> D(i+1,j+1) <
//    D(i,j); Del <=> D(i+1,j) < D(i,j); else Ins.
//  * TB walks those codes from (0,0) in lock step across the lanes that
//    solved their window. A final window wider than C continues as a new
//    DC segment on the untouched suffix (suffix distances are intrinsic).
#pragma once

#include <cstdint>

#include <vector_types.h>

namespace sgk {

// Per-pair status (low 16 bits = kind as the C ABI's SG_* codes, high = detail).
enum : int32_t {
    kStOk = 0,
    kStInternal = 3,
    kDetBudgetI = 1 << 16,      // traceback.cpp:76-78
    kDetBudgetD = 2 << 16,      // traceback.cpp:84-86
    kDetLeftover = 3 << 16,     // traceback.cpp:110-111
    kDetWatchdog = 4 << 16,     // aligner.cpp:81-82
    kDetNoStep = 5 << 16,       // traceback.cpp:105-106
    kDetSegment = 6 << 16,      // continuation segment disagrees with the budget
};

struct AlignParams {
    const uint32_t* seq;      // 2-bit packed bases, 16 per word, base k at bits 2(k%16)
    const uint32_t* nmask;    // 1 bit per base (same base offsets), may be null
    const int64_t* text_off;  // base offset of each text
    const int64_t* pat_off;   // base offset of each pattern
    const int32_t* text_len;
    const int32_t* pat_len;
    const uint8_t* has_n;     // per pair: any non-ACGT base (may be null)
    const int32_t* order;     // processing order (null = identity)
    int32_t n_pairs;
    const int32_t* n_fresh;   // device count of the pairs in `order` to take (null: n_pairs)
    int32_t W, O, et, policy; // policy: 0 BaselineEdges, 1 SeneEntries, 2 DentTrimmed (counters)
    int32_t two;              // the constant 2 at run time (keeps the DP shift an IMAD)
    int32_t single;           // single-window mode (aligner.cpp:87-112)
    int32_t k_single;         // its edit budget
    // outputs
    int32_t* distance;
    int32_t* windows;
    int32_t* status;
    int32_t* out_bytes;       // run bytes per pair
    uint64_t* counters;       // [n_pairs][7] (InstrumentationCounters order) or null
    const int64_t* bound_off; // byte offset (4-aligned) of each pair's run region in scratch
    uint32_t* scratch;        // run bytes, (op << 6) | (len - 1)
    uint32_t* bnd;            // parked rows: per warp [32L + 5 slots][32 lanes][L]
    const uint32_t* bnd_ones;   // one warp's worth of parked-row slots holding ones / zeros,
    const uint32_t* bnd_zeros;  // read in a window's first chunk / by an idle lane
    unsigned int* next_pair;  // work queue head
    const unsigned int* ready;  // [n_chunks] sequence-word chunk has arrived (streamed upload)
    int64_t chunk_words;
    int32_t n_chunks;
    int32_t wcap;             // K6: widest window (columns) a warp's scratch holds
    // K1 mixed: band warps (K1b) <-> full-frame warps
    int32_t mixed;
    int32_t band_active;      // band warps that take pairs (spread over the blocks)
    int32_t band_subchunks;   // band chunks per phase (0: the default, 16 rows)
    uint32_t* q_band;         // pairs handed to band warps: [32 + n_pairs] (head, tail, slots)
    uint32_t* q_full;         // pairs handed to full-frame warps
    uint32_t* q_coop;         // pairs handed to the cooperative warps (one window per warp)
    uint32_t* q_std;          // pairs whose next window the STD frame takes (m_w <= 31)
    unsigned int* remaining;  // pairs not finished (warps exit at 0)
    int32_t* resume_state;    // [n_pairs][4]: toff, poff, cur_op | cur_len << 8, open word
    int32_t* u_list;          // K0 (§3.10): pairs left to a full-frame K1 launch after the
    unsigned int* u_count;    // mixed one (unrelated pairs and every pair's tail windows)
    int32_t restore;          // the fresh pairs resume from resume_state (that launch)
    int32_t* t_list;          // pairs whose next window is an STD window (m_w <= 31, the
    unsigned int* t_count;    // pattern all but consumed): the tail K1 (k1_tail) after K1 mixed
    unsigned int* coop_out;   // pairs a band warp handed to a cooperative warp and not yet
                              // taken back (in q_coop, at a cooperative warp, or in q_band)
    // finished-pair counts per output slice (one-shot calls): a pair's run bytes and
    // counts are complete when its slice's count includes it (null: no slices)
    unsigned int* slice_done;
    int32_t slice_pairs;      // pairs per slice (pair k is in slice k / slice_pairs)
    // pipelined launches (§3.12): K1 mixed on most SMs, the tail / full-frame K1 of each
    // output slice beside it on the SMs it leaves free. K1 mixed: t_list / u_list hold one
    // region of slice_pairs entries per slice, t_count / u_count one count per slice, and
    // body_done[sl] counts the pairs of slice sl that have left it (null: one list each).
    // The tail K1 of a slice starts once *wait_count >= wait_target (null: at once).
    unsigned int* body_done;
    int32_t last_slice;       // pairs from last_slice * slice_pairs on are one slice
    const unsigned int* wait_count;
    unsigned int wait_target;
    unsigned int* pipe_err;   // set when such a wait timed out (the host fails the call)
    unsigned long long* phase_cycles;  // optional [8]: phase cycles and counts (diagnostics)
    unsigned long long* warp_times;    // optional [warps][2]: start / exit globaltimer, smid (diagnostics)
};

// Launch K1 for limb count L (W <= 32L). Returns cudaError_t as int.
int launch_window_align(int L, const AlignParams& p, int grid, int warps_per_block,
                        void* stream);
// Bytes of parked-row scratch needed for `total_warps` warps at limb count L.
size_t bnd_scratch_bytes(int L, long long total_warps);
// Shared memory per block and the warps per block used for L.
int k1_warps_per_block(int L);
size_t k1_smem_bytes(int L);
int k1_max_blocks_per_sm(int L);

// K6 (csrc/wide_align.cu): one warp per pair, for windows wider than 128 bits
// (W <= 1024, single windows <= 1024 characters). Scratch per warp, in words:
// parked row and its shift [wcap + 16][L] each, traceback events X and Y
// [wcap + 8][L] each, L = ceil(wcap / 32) limbs.
#ifdef __CUDACC__
__host__ __device__
#endif
inline long long wide_warp_words(int wcap) {  // 128-byte multiple
    return ((4LL * ((wcap + 3) & ~3) + 48) * ((wcap + 31) / 32) + 31) & ~31LL;
}
int launch_wide_align(const AlignParams& p, int grid, void* stream);
int wide_warps_per_block();
size_t wide_smem_bytes();
int wide_max_blocks_per_sm();

// K1 mixed: one persistent block per SM of band warps (K1b,
// windows of W <= 64 columns in diagonal coordinates) and full-frame warps
// (limb count LF); pairs move between them through device queues.
int launch_mixed_align(int LF, const AlignParams& p, int grid, void* stream);
// The tail K1 (§3.10): band-type warps resume the pairs of p.order (their STD windows,
// the standard single-word frame); any other window goes to p.u_list.
int launch_tail_align(const AlignParams& p, int grid, void* stream);
int launch_queue_init(uint32_t* q_band, uint32_t* q_full, uint32_t* q_coop, uint32_t* q_std,
                      unsigned* remaining, int n, const int32_t* n_dev, void* stream);

int mixed_band_warps();
int mixed_full_warps();
int mixed_warps_per_block();  // band + full-frame + cooperative warps
int mixed_max_blocks_per_sm(int LF);
bool band_eligible(int W, int O, int single);

// K7 (csrc/exact_align.cu): optimal global alignment with the reference
// oracle's tie-breaking (proj/src/oracle.cpp:39-89), one warp per pair.
struct ExactParams {
    const uint32_t* seq;       // as AlignParams
    const uint32_t* nmask;
    const int64_t* text_off;
    const int64_t* pat_off;
    const int32_t* text_len;
    const int32_t* pat_len;
    const uint8_t* has_n;
    int32_t n_pairs;
    uint4* store;              // per pair [ceil(m/32)][n] x (Pv, Mv, Ph, Mh)
    const int64_t* store_off;  // in uint4 units
    int8_t* hbuf;              // per pair: bottom carries between 1024-row stripes
    const int64_t* hbuf_off;   // bytes, 16-aligned, >= roundup16(n) + 16 per pair
    const int64_t* bound_off;  // run-byte region of each pair (as K1)
    uint8_t* scratch;
    int32_t* distance;
    int32_t* out_bytes;
};
int launch_exact_align(const ExactParams& p, void* stream);

// K2/K3: exclusive scan of the per-pair run byte counts (dense_off has n+1
// entries, the total last) and compaction of the bounded run regions into one
// dense byte buffer.
int launch_cigar_offsets(const int32_t* out_bytes, int64_t* dense_off, int32_t n, void* temp,
                         size_t temp_bytes, void* stream);
size_t cigar_offsets_temp_bytes(int32_t n);
int launch_cigar_compact(const uint32_t* scratch, const int64_t* bound_off,
                         const int64_t* dense_off, const int32_t* out_bytes, uint8_t* dense,
                         int32_t n, void* stream);
// K2/K3 per output slice [lo, hi) while K1 still runs (one-shot calls, on a second
// stream): waits until the slice's pairs have all finished (slice_done[s] == hi - lo),
// scans their run byte counts onto the running offset (dense_off[lo] holds the
// previous slices' total; dense_off[hi] receives the new one), compacts their bytes,
// and reports (first byte, bytes) of the slice in info[2s], info[2s + 1] (host-mapped).
int launch_slice_scan(const int32_t* out_bytes, int64_t* dense_off, int32_t lo, int32_t hi,
                      const unsigned* slice_done, int s, int64_t* info, void* stream);
int launch_slice_compact(const uint32_t* scratch, const int64_t* bound_off,
                         const int64_t* dense_off, const int32_t* out_bytes, uint8_t* dense,
                         int32_t lo, int32_t hi, void* stream);

}  // namespace sgk
