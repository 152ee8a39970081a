/*
 * Seeded synthetic read/reference pairs for the BASELINE.json configs.
 *
 * The reference ships its own simulator (proj/src/simulate.cpp:12-70,
 * Bernoulli per-position errors, no text slack). The benchmark configs need
 * exact edit counts, text slack, indel mixes and uncorrelated pairs, so this
 * generator is new. It keeps the reference's RNG:
 * SplitMix64 (proj/include/scrooge/rng.hpp:10-30), so a (spec, pair index)
 * reproduces the same pair on every host and thread count.
 *
 * Per pair p (all draws from SplitMix64(pair_seed(seed, p)), in this order):
 *   1. read length L: fixed, or log-uniform in [read_min, read_max];
 *   2. uncorrelated flag (only when frac_uncorrelated > 0);
 *   3. uncorrelated: text = L iid bases, pattern = L iid bases;
 *      correlated: text = L + slack iid bases, rate ~ U[rate_min, rate_max],
 *      E = round(rate * L) distinct edit positions in [0, L) (Floyd sampling),
 *      each typed sub/ins/del by the mix; pattern = text[0:L) with the edits
 *      applied (sub = a different base, ins = a random base placed before the
 *      position, del = drop the position).
 * Bases are 2-bit codes A=0 C=1 G=2 T=3 (proj/include/scrooge/sequence.hpp:13-27).
 */
#ifndef SG_SYNTH_H
#define SG_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sg_synth_spec {
    int64_t n_pairs;
    uint64_t seed;
    int32_t read_min, read_max;   /* equal => fixed read length */
    int32_t slack_abs;            /* text = read + slack_abs + round(slack_frac*read) */
    double slack_frac;
    double rate_min, rate_max;    /* per-pair edit rate, uniform in [min, max] */
    double mix_sub, mix_ins, mix_del;
    double frac_uncorrelated;     /* fraction of independent equal-length pairs */
} sg_synth_spec;

/* SplitMix64 step and the p-th output of SplitMix64(seed) in O(1). */
uint64_t sg_splitmix_next(uint64_t* state);
uint64_t sg_pair_seed(uint64_t seed, int64_t p);

/* Upper bounds on text / pattern length for any pair of the spec. */
int64_t sg_synth_max_text(const sg_synth_spec* spec);
int64_t sg_synth_max_pattern(const sg_synth_spec* spec);

/* Generates pair p as 1-byte codes. Buffers must hold sg_synth_max_text /
 * sg_synth_max_pattern codes. Returns 0, or -1 on a bad spec. */
int sg_synth_pair(const sg_synth_spec* spec, int64_t p, uint8_t* text, int64_t* n,
                  uint8_t* pattern, int64_t* m);

/* The five BASELINE.json configs (1-based id; 0 = invalid). cfg4's (W, O)
 * sweep shares one pair set. */
int sg_synth_baseline_spec(int cfg_id, sg_synth_spec* out);

#ifdef __cplusplus
}
#endif

#endif
