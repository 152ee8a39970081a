/* Seeded synthetic pairs; see synth.h for the generation rules. */
#include "synth.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define SM_GAMMA 0x9E3779B97F4A7C15ull

static uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t sg_splitmix_next(uint64_t* state) { return sm_mix(*state += SM_GAMMA); }

uint64_t sg_pair_seed(uint64_t seed, int64_t p) {
    return sm_mix(seed + (uint64_t)(p + 1) * SM_GAMMA);
}

/* next_below / next_unit as in proj/include/scrooge/rng.hpp:23-26 */
static uint64_t below(uint64_t* s, uint64_t n) { return sg_splitmix_next(s) % n; }
static double unit(uint64_t* s) { return (double)(sg_splitmix_next(s) >> 11) * 0x1.0p-53; }

static void random_bases(uint64_t* s, uint8_t* out, int64_t len) {
    uint64_t w = 0;
    for (int64_t i = 0; i < len; ++i) {
        if ((i & 31) == 0) w = sg_splitmix_next(s);
        out[i] = (uint8_t)(w & 3);
        w >>= 2;
    }
}

static int64_t slack_of(const sg_synth_spec* spec, int64_t L) {
    return (int64_t)spec->slack_abs + (int64_t)llround(spec->slack_frac * (double)L);
}

int64_t sg_synth_max_text(const sg_synth_spec* spec) {
    return (int64_t)spec->read_max + slack_of(spec, spec->read_max) + 1;
}

int64_t sg_synth_max_pattern(const sg_synth_spec* spec) { return 2 * (int64_t)spec->read_max + 1; }

int sg_synth_pair(const sg_synth_spec* spec, int64_t p, uint8_t* text, int64_t* n,
                  uint8_t* pattern, int64_t* m) {
    if (spec->read_min < 1 || spec->read_max < spec->read_min) return -1;
    uint64_t s = sg_pair_seed(spec->seed, p);
    int64_t L = spec->read_min;
    if (spec->read_max > spec->read_min) {
        const double lo = log((double)spec->read_min), hi = log((double)spec->read_max);
        L = (int64_t)llround(exp(lo + unit(&s) * (hi - lo)));
        if (L < spec->read_min) L = spec->read_min;
        if (L > spec->read_max) L = spec->read_max;
    }
    int uncorrelated = 0;
    if (spec->frac_uncorrelated > 0) uncorrelated = unit(&s) < spec->frac_uncorrelated;
    if (uncorrelated) {
        random_bases(&s, text, L);
        random_bases(&s, pattern, L);
        *n = L;
        *m = L;
        return 0;
    }
    const int64_t nt = L + slack_of(spec, L);
    random_bases(&s, text, nt);
    double rate = spec->rate_min;
    if (spec->rate_max > spec->rate_min) rate += unit(&s) * (spec->rate_max - spec->rate_min);
    int64_t E = (int64_t)llround(rate * (double)L);
    if (E > L) E = L;
    if (E < 0) E = 0;
    /* Floyd's sampling of E distinct positions into a bitmap */
    const int64_t words = (L + 63) / 64;
    uint64_t stack_bits[64];
    uint64_t* bits = words <= 64 ? stack_bits : (uint64_t*)calloc((size_t)words, 8);
    if (!bits) return -1;
    memset(bits, 0, (size_t)words * 8);
    for (int64_t j = L - E; j < L; ++j) {
        const int64_t t = (int64_t)below(&s, (uint64_t)j + 1);
        if (bits[t >> 6] >> (t & 63) & 1)
            bits[j >> 6] |= 1ull << (j & 63);
        else
            bits[t >> 6] |= 1ull << (t & 63);
    }
    const double c_sub = spec->mix_sub, c_ins = spec->mix_sub + spec->mix_ins;
    int64_t k = 0;
    for (int64_t i = 0; i < L; ++i) {
        if (bits[i >> 6] >> (i & 63) & 1) {
            const double u = unit(&s);
            if (u < c_sub) {
                pattern[k++] = (uint8_t)((text[i] + 1 + below(&s, 3)) & 3);
            } else if (u < c_ins) {
                pattern[k++] = (uint8_t)below(&s, 4);
                pattern[k++] = text[i];
            } /* else: deletion drops text[i] */
        } else {
            pattern[k++] = text[i];
        }
    }
    if (bits != stack_bits) free(bits);
    if (k == 0) pattern[k++] = (uint8_t)((text[0] + 1) & 3);
    *n = nt;
    *m = k;
    return 0;
}

int sg_synth_baseline_spec(int cfg_id, sg_synth_spec* o) {
    memset(o, 0, sizeof *o);
    o->mix_sub = o->mix_ins = o->mix_del = 1.0 / 3;
    switch (cfg_id) {
        case 1: /* short plumbing: 100 bp reads, 10 bp slack, 5%, 1:1:1 */
            o->n_pairs = 10000; o->seed = 1; o->read_min = o->read_max = 100;
            o->slack_abs = 10; o->rate_min = o->rate_max = 0.05;
            return 1;
        case 2: /* Illumina-like: 250 bp, +20 bp slack, 2%, 8:1:1 */
            o->n_pairs = 1000000; o->seed = 2; o->read_min = o->read_max = 250;
            o->slack_abs = 20; o->rate_min = o->rate_max = 0.02;
            o->mix_sub = 0.8; o->mix_ins = 0.1; o->mix_del = 0.1;
            return 2;
        case 3: /* long noisy: 10 kbp, +5% slack, 15%, 2:5:3 */
            o->n_pairs = 100000; o->seed = 3; o->read_min = o->read_max = 10000;
            o->slack_frac = 0.05; o->rate_min = o->rate_max = 0.15;
            o->mix_sub = 0.2; o->mix_ins = 0.5; o->mix_del = 0.3;
            return 3;
        case 4: /* W/O sweep: 10 kbp, no slack, 10%, 1:1:1 */
            o->n_pairs = 20000; o->seed = 4; o->read_min = o->read_max = 10000;
            o->rate_min = o->rate_max = 0.10;
            return 4;
        case 5: /* mixed: log-uniform 100..20000, 70% correlated 5-15%, 30% independent */
            o->n_pairs = 500000; o->seed = 5; o->read_min = 100; o->read_max = 20000;
            o->slack_frac = 0.05; o->rate_min = 0.05; o->rate_max = 0.15;
            o->frac_uncorrelated = 0.30;
            return 5;
        default:
            return 0;
    }
}
