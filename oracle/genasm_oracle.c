/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see genasm_oracle.h).
 *
 * CPU restatement of the reference windowed GenASM path. Bit vectors follow
 * proj/include/scrooge/bitvec.hpp:13-24: bit j = 0 is the MSB of word 0, a
 * DP shift moves bits toward j = 0 and the bit entering at j = m-1 is the
 * explicit end-of-pattern boundary (proj/include/scrooge/dp.hpp:145-154).
 */
#include "genasm_oracle.h"

#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_BITS 1024                 /* BitVector::kMaxBits, bitvec.hpp:29 */
#define ORC_MAX_WORDS (ORC_MAX_BITS / 64) /* BitVector::kMaxWords */

typedef uint64_t word;

static int fail(char* err, size_t errlen, int code, const char* fmt, ...) {
    if (err && errlen) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err, errlen, fmt, ap);
        va_end(ap);
    }
    return code;
}

/* ---- per-thread window statistics (design studies only) ---- */
static __thread int32_t* st_dopt;
static __thread int32_t* st_nw;
static __thread int32_t* st_mw;
static __thread int64_t st_len, st_cap;

static void stats_push(int32_t d, int32_t nw, int32_t mw) {
    if (st_len == st_cap) {
        st_cap = st_cap ? 2 * st_cap : 1024;
        st_dopt = (int32_t*)realloc(st_dopt, (size_t)st_cap * 4);
        st_nw = (int32_t*)realloc(st_nw, (size_t)st_cap * 4);
        st_mw = (int32_t*)realloc(st_mw, (size_t)st_cap * 4);
    }
    st_dopt[st_len] = d;
    st_nw[st_len] = nw;
    st_mw[st_len] = mw;
    ++st_len;
}

int64_t orc_last_window_count(void) { return st_len; }

void orc_last_window_stats(int32_t* d_opt, int32_t* n_w, int32_t* m_w, int64_t cap) {
    for (int64_t w = 0; w < st_len && w < cap; ++w) {
        if (d_opt) d_opt[w] = st_dopt[w];
        if (n_w) n_w[w] = st_nw[w];
        if (m_w) m_w[w] = st_mw[w];
    }
}

/* ---- growable CIGAR (cigar_append, proj/src/cigar.cpp:9-16) ---- */
typedef struct {
    char* ops;
    int64_t* lens;
    int64_t n, cap;
} cigar_t;

static void cigar_append(cigar_t* c, char op, int64_t len) {
    if (len <= 0) return;
    if (c->n && c->ops[c->n - 1] == op) {
        c->lens[c->n - 1] += len;
        return;
    }
    if (c->n == c->cap) {
        c->cap = c->cap ? 2 * c->cap : 16;
        c->ops = (char*)realloc(c->ops, (size_t)c->cap);
        c->lens = (int64_t*)realloc(c->lens, (size_t)c->cap * 8);
    }
    c->ops[c->n] = op;
    c->lens[c->n] = len;
    ++c->n;
}

/* ---- one window's DP table R[i][d], i = 0..n, d = 0..rows-1 (untrimmed) ---- */
typedef struct {
    int n, m, k, wpv;
    int rows;        /* rows computed (= rows stored) */
    word* r;         /* r[((size_t)d * (n + 1) + i) * wpv + w] */
    size_t cap;      /* words allocated */
    word pm[5][ORC_MAX_WORDS];
} window_t;

static word* entry(window_t* t, int i, int d) {
    return t->r + ((size_t)d * (size_t)(t->n + 1) + (size_t)i) * (size_t)t->wpv;
}

static int bit_of(const word* v, int j) { return (int)((v[j >> 6] >> (63 - (j & 63))) & 1u); }

/* build_pattern_masks, proj/src/dp.cpp:8-21 (+ match_nothing for text N) */
static void build_masks(window_t* t, const uint8_t* p) {
    const int m = t->m, wpv = t->wpv;
    for (int c = 0; c < 5; ++c) {
        for (int w = 0; w < wpv; ++w) t->pm[c][w] = ~(word)0;
        const int used = m % 64;
        if (used) t->pm[c][wpv - 1] &= ~(word)0 << (64 - used);
    }
    for (int j = 0; j < m; ++j)
        if (p[j] < 4) t->pm[p[j]][j >> 6] &= ~((word)1 << (63 - (j & 63)));
}

static int grow_rows(window_t* t, int rows) {
    const size_t need = (size_t)rows * (size_t)(t->n + 1) * (size_t)t->wpv;
    if (need <= t->cap) return 0;
    size_t cap = t->cap ? t->cap : 4096;
    while (cap < need) cap *= 2;
    word* r = (word*)realloc(t->r, cap * sizeof(word));
    if (!r) return -1;
    t->r = r;
    t->cap = cap;
    return 0;
}

/* compute_dc, proj/src/dp.cpp:104-231. Returns d_opt or -1. */
static int compute_dc(window_t* t, const uint8_t* text, int et) {
    const int n = t->n, m = t->m, k = t->k, wpv = t->wpv, last = wpv - 1;
    const word end_bit = (word)1 << (63 - ((m - 1) % 64));
    int found = -1;
    if (grow_rows(t, 1)) return -2;
    /* row 0: init column, then the exact-match rule (dp.cpp:145-172) */
    word* init = entry(t, n, 0);
    for (int w = 0; w < wpv; ++w) init[w] = t->pm[4][w]; /* ones(m) */
    for (int i = n - 1; i >= 0; --i) {
        const word* right = entry(t, i + 1, 0);
        word* out = entry(t, i, 0);
        const word* pm = t->pm[text[i] < 4 ? text[i] : 4];
        for (int w = 0; w < wpv; ++w) {
            const word carry = w < last ? right[w + 1] >> 63 : 0;
            out[w] = ((right[w] << 1) | carry) | pm[w];
        }
        if (n - i - 1 > 0) out[last] |= end_bit;
    }
    t->rows = 1;
    if ((entry(t, 0, 0)[0] >> 63) == 0) found = 0;
    /* rows d = 1..k (dp.cpp:176-223) */
    for (int d = 1; d <= k; ++d) {
        if (found >= 0 && et) break;
        if (grow_rows(t, d + 1)) return -2;
        /* init column: ones(m).shl(min(d, m)) */
        word* col = entry(t, n, d);
        const int s = d < m ? d : m;
        for (int w = 0; w < wpv; ++w) col[w] = 0;
        if (s < m) {
            const word* ones = t->pm[4];
            const int off = s / 64, sh = s % 64;
            for (int w = 0; w + off < wpv; ++w) {
                word x = ones[w + off] << sh;
                if (sh && w + off + 1 < wpv) x |= ones[w + off + 1] >> (64 - sh);
                col[w] = x;
            }
            const int used = m % 64;
            if (used) col[last] &= ~(word)0 << (64 - used);
        }
        for (int i = n - 1; i >= 0; --i) {
            const word* north = entry(t, i, d - 1);
            const word* diag = entry(t, i + 1, d - 1);
            const word* east = entry(t, i + 1, d);
            word* out = entry(t, i, d);
            const word* pm = t->pm[text[i] < 4 ? text[i] : 4];
            const word end_ins = n - i <= d - 1 ? 0 : end_bit;
            const word end_sub = n - i - 1 <= d - 1 ? 0 : end_bit;
            const word end_mat = n - i - 1 <= d ? 0 : end_bit;
            for (int w = 0; w < wpv; ++w) {
                const word cn = w < last ? north[w + 1] >> 63 : 0;
                const word cd = w < last ? diag[w + 1] >> 63 : 0;
                const word ce = w < last ? east[w + 1] >> 63 : 0;
                word ins = (north[w] << 1) | cn;
                word sub = (diag[w] << 1) | cd;
                word mat = ((east[w] << 1) | ce) | pm[w];
                if (w == last) {
                    ins |= end_ins;
                    sub |= end_sub;
                    mat |= end_mat;
                }
                out[w] = ins & diag[w] & sub & mat;
            }
        }
        t->rows = d + 1;
        if (found < 0 && (entry(t, 0, d)[0] >> 63) == 0) found = d;
    }
    return found;
}

/* Edge bit j of cell (i, d), regenerated from entries: regen_edges,
 * proj/src/traceback.cpp:35-54 (Baseline policy stores the same edges,
 * traceback.cpp:15-31, proj/tests/test_traceback.cpp:94-116). */
typedef struct {
    int mat, sub, del, ins;
} edge_bits;

static edge_bits edges_at(window_t* t, int i, int d, int j, uint8_t tc) {
    const int n = t->n, m = t->m;
    const word* pm = t->pm[tc < 4 ? tc : 4];
    edge_bits e;
    if (d == 0) {
        e.ins = e.del = e.sub = 1;
        const int shifted = j + 1 < m ? bit_of(entry(t, i + 1, 0), j + 1) : (n - i - 1 > 0);
        e.mat = shifted | bit_of(pm, j);
        return e;
    }
    e.ins = j + 1 < m ? bit_of(entry(t, i, d - 1), j + 1) : (n - i > d - 1);
    e.del = bit_of(entry(t, i + 1, d - 1), j);
    e.sub = j + 1 < m ? bit_of(entry(t, i + 1, d - 1), j + 1) : (n - i - 1 > d - 1);
    e.mat = (j + 1 < m ? bit_of(entry(t, i + 1, d), j + 1) : (n - i - 1 > d)) | bit_of(pm, j);
    return e;
}

typedef struct {
    int text_consumed, pattern_consumed, cost, nops;
} transcript_t;

/* traceback, proj/src/traceback.cpp:56-113. Ops appended to `c`. */
static int traceback(window_t* t, int d_opt, const uint8_t* text, int max_steps, cigar_t* c,
                     transcript_t* ts, uint64_t* reads, char* err, size_t errlen) {
    const int n = t->n, m = t->m;
    if (d_opt < 0 || d_opt > t->k || d_opt >= t->rows)
        return fail(err, errlen, ORC_INTERNAL, "traceback: d_opt %d not covered by the stored table",
                    d_opt);
    int i = 0, j = 0, d = d_opt;
    memset(ts, 0, sizeof *ts);
    while (max_steps < 0 || ts->nops < max_steps) {
        char op;
        if (i == n && j == m) break;
        if (i == n) {
            if (d != m - j)
                return fail(err, errlen, ORC_INTERNAL, "traceback: budget %d != remaining pattern %d",
                            d, m - j);
            op = 'I';
        } else if (j == m) {
            if (d != n - i)
                return fail(err, errlen, ORC_INTERNAL, "traceback: budget %d != remaining text %d", d,
                            n - i);
            op = 'D';
        } else {
            *reads += d == 0 ? 1 : 3;
            const edge_bits e = edges_at(t, i, d, j, text[i]);
            if (!e.mat)
                op = '=';
            else if (d > 0 && !e.sub)
                op = 'X';
            else if (d > 0 && !e.del)
                op = 'D';
            else if (d > 0 && !e.ins)
                op = 'I';
            else
                return fail(err, errlen, ORC_INTERNAL,
                            "traceback: no legal step at (i=%d, j=%d, d=%d)", i, j, d);
        }
        switch (op) {
            case '=': ++i, ++j; break;
            case 'X': ++i, ++j, --d; break;
            case 'D': ++i, --d; break;
            default: ++j, --d; break;
        }
        cigar_append(c, op, 1);
        ts->nops += 1;
        if (op != '=') ts->cost += 1;
        ts->text_consumed += (op == '=' || op == 'X' || op == 'D');
        ts->pattern_consumed += (op == '=' || op == 'X' || op == 'I');
    }
    if (max_steps < 0 && d != 0)
        return fail(err, errlen, ORC_INTERNAL, "traceback: finished with leftover budget %d", d);
    return ORC_OK;
}

enum policy { POL_BASELINE, POL_SENE, POL_DENT };

/* Counter arithmetic of DpTable stores, proj/src/dp.cpp:23-37,58-75,225-228. */
static void dc_counters(orc_counters* c, enum policy pol, int n, int m, int k, int rows,
                        int tl) {
    int keep_cols = n + 1, keep_bits = m;
    if (pol == POL_DENT) {
        keep_cols = (n < tl ? n : tl) + 1;
        keep_bits = m < tl + 1 ? m : tl + 1;
    }
    const uint64_t slots = pol == POL_BASELINE ? 3 : 1;
    c->stored_bits += (uint64_t)rows * (uint64_t)keep_cols * (uint64_t)keep_bits * slots;
    c->table_writes += (uint64_t)rows * (uint64_t)keep_cols * slots;
    c->cells_computed += (uint64_t)rows * (uint64_t)n;
    c->rows_computed += (uint64_t)rows;
    c->rows_possible += (uint64_t)k + 1;
    c->baseline_equiv_bits += 3ull * ((uint64_t)n + 1) * ((uint64_t)k + 1) * (uint64_t)m;
}

/* AlignerConfig::validate, proj/src/aligner.cpp:8-18 */
static int validate(const orc_config* cfg, char* err, size_t errlen) {
    if (cfg->W < 1 || cfg->W > ORC_MAX_BITS)
        return fail(err, errlen, ORC_CONFIG, "window size W out of range: %d", cfg->W);
    if (cfg->O < 0 || cfg->O >= cfg->W)
        return fail(err, errlen, ORC_CONFIG,
                    "window overlap O must satisfy 0 <= O < W, got O=%d W=%d", cfg->O, cfg->W);
    if (cfg->dent && cfg->single_window)
        return fail(err, errlen, ORC_CONFIG,
                    "trimmed table storage cannot back a full single-window traceback");
    if (cfg->single_window && (cfg->k_single < 0 || cfg->k_single > ORC_MAX_BITS))
        return fail(err, errlen, ORC_CONFIG, "k out of range: %d", cfg->k_single);
    return ORC_OK;
}

static int finish(orc_result* out, cigar_t* c, int rc) {
    if (rc != ORC_OK) {
        free(c->ops);
        free(c->lens);
        out->ops = NULL;
        out->lens = NULL;
        out->n_runs = 0;
        return rc;
    }
    out->ops = c->ops;
    out->lens = c->lens;
    out->n_runs = c->n;
    return ORC_OK;
}

static int align_single(const orc_config* cfg, const uint8_t* text, int64_t n,
                        const uint8_t* pattern, int64_t m, orc_result* out, char* err,
                        size_t errlen) {
    /* align_single_window, proj/src/aligner.cpp:87-112 (validation order kept) */
    if (n == 0 || m == 0) return fail(err, errlen, ORC_INPUT, "align: empty input sequence");
    if (cfg->dent)
        return fail(err, errlen, ORC_CONFIG,
                    "trimmed table storage cannot back a full single-window traceback");
    if (n > ORC_MAX_BITS || m > ORC_MAX_BITS)
        return fail(err, errlen, ORC_CONFIG,
                    "single-window mode requires sequences of at most 1024 characters");
    if (cfg->k_single < 0 || cfg->k_single > ORC_MAX_BITS)
        return fail(err, errlen, ORC_CONFIG, "compute_dc: k out of range: %d", cfg->k_single);
    window_t t;
    memset(&t, 0, sizeof t);
    t.n = (int)n;
    t.m = (int)m;
    t.k = cfg->k_single;
    t.wpv = (t.m + 63) / 64;
    build_masks(&t, pattern);
    const int d_opt = compute_dc(&t, text, cfg->et);
    cigar_t c = {0};
    out->windows = 1;
    dc_counters(&out->counters, cfg->sene ? POL_SENE : POL_BASELINE, t.n, t.m, t.k, t.rows, -1);
    stats_push(d_opt, t.n, t.m);
    if (d_opt == -2) {
        free(t.r);
        return fail(err, errlen, ORC_INTERNAL, "out of memory");
    }
    if (d_opt < 0) {
        free(t.r);
        out->found = 0;
        out->distance = -1;
        return finish(out, &c, ORC_OK);
    }
    transcript_t ts;
    uint64_t reads = 0;
    /* counters were added before traceback (aligner.cpp:98-99): TB reads are not reported */
    int rc = traceback(&t, d_opt, text, -1, &c, &ts, &reads, err, errlen);
    free(t.r);
    if (rc == ORC_OK && (ts.text_consumed != t.n || ts.pattern_consumed != t.m))
        rc = fail(err, errlen, ORC_INTERNAL, "single-window traceback did not consume both sequences");
    out->found = 1;
    out->distance = ts.cost;
    return finish(out, &c, rc);
}

int orc_align(const orc_config* cfg, const uint8_t* text, int64_t n, const uint8_t* pattern,
              int64_t m, orc_result* out, char* err, size_t errlen) {
    memset(out, 0, sizeof *out);
    st_len = 0;
    int rc = validate(cfg, err, errlen);
    if (rc) return rc;
    if (cfg->single_window) return align_single(cfg, text, n, pattern, m, out, err, errlen);
    if (n == 0 || m == 0) return fail(err, errlen, ORC_INPUT, "align: empty input sequence");

    const int W = cfg->W;
    const int step_limit = W - cfg->O;
    const int64_t window_cap = 4 * ((n + m) / step_limit + 2); /* aligner.cpp:40 */
    const enum policy base_pol = cfg->dent ? POL_DENT : cfg->sene ? POL_SENE : POL_BASELINE;
    cigar_t c = {0};
    window_t t;
    memset(&t, 0, sizeof t);
    int64_t toff = 0, poff = 0;
    out->found = 1;
    for (;;) {
        const int64_t n_rem = n - toff, m_rem = m - poff;
        if (n_rem == 0 && m_rem == 0) break;
        if (n_rem == 0) { /* aligner.cpp:48-52 */
            cigar_append(&c, 'I', m_rem);
            out->distance += m_rem;
            break;
        }
        if (m_rem == 0) { /* aligner.cpp:53-57 */
            cigar_append(&c, 'D', n_rem);
            out->distance += n_rem;
            break;
        }
        const int final_window = n_rem <= W && m_rem <= W;
        t.n = (int)(n_rem < W ? n_rem : W);
        t.m = (int)(m_rem < W ? m_rem : W);
        t.k = W;
        t.wpv = (t.m + 63) / 64;
        enum policy pol = base_pol;
        if (final_window && pol == POL_DENT) pol = POL_SENE; /* aligner.cpp:62-64 */
        build_masks(&t, pattern + poff);
        const int d_opt = compute_dc(&t, text + toff, cfg->et);
        if (d_opt == -2) {
            rc = fail(err, errlen, ORC_INTERNAL, "out of memory");
            break;
        }
        if (d_opt < 0) {
            rc = fail(err, errlen, ORC_INTERNAL,
                      "windowed alignment: no distance <= W found in a window");
            break;
        }
        stats_push(d_opt, t.n, t.m);
        dc_counters(&out->counters, pol, t.n, t.m, t.k, t.rows, step_limit);
        transcript_t ts;
        uint64_t reads = 0;
        rc = traceback(&t, d_opt, text + toff, final_window ? -1 : step_limit, &c, &ts, &reads,
                       err, errlen);
        out->counters.table_reads += reads;
        if (rc) break;
        if (ts.nops == 0) {
            rc = fail(err, errlen, ORC_INTERNAL, "windowed alignment: window made no progress");
            break;
        }
        out->distance += ts.cost;
        toff += ts.text_consumed;
        poff += ts.pattern_consumed;
        out->windows += 1;
        if (out->windows > window_cap) {
            rc = fail(err, errlen, ORC_INTERNAL,
                      "windowed alignment: window count exceeded watchdog cap");
            break;
        }
    }
    free(t.r);
    return finish(out, &c, rc);
}

void orc_result_free(orc_result* r) {
    free(r->ops);
    free(r->lens);
    r->ops = NULL;
    r->lens = NULL;
    r->n_runs = 0;
}

int64_t orc_cigar_string(const orc_result* r, char* buf, int64_t cap) {
    int64_t pos = 0;
    char tmp[32];
    for (int64_t k = 0; k < r->n_runs; ++k) {
        const int len = snprintf(tmp, sizeof tmp, "%lld%c", (long long)r->lens[k], r->ops[k]);
        if (buf && pos + len < cap) memcpy(buf + pos, tmp, (size_t)len);
        pos += len;
    }
    if (buf && pos < cap) buf[pos] = '\0';
    return pos;
}

/* ---- replay checks (test-side; proj/src/cigar.cpp:70-107) ---- */
static int bases_match(uint8_t a, uint8_t b) { return a == b && a < 4; }

int64_t orc_replay_runs(const uint8_t* text, int64_t n, const uint8_t* pattern, int64_t m,
                        const uint8_t* runs, int64_t nbytes) {
    int64_t i = 0, j = 0, edits = 0;
    for (int64_t b = 0; b < nbytes; ++b) {
        const int op = runs[b] >> 6;
        const int64_t len = (runs[b] & 63) + 1;
        for (int64_t r = 0; r < len; ++r) {
            switch (op) {
                case 0:
                    if (i >= n || j >= m || !bases_match(text[i], pattern[j])) return -1;
                    ++i, ++j;
                    break;
                case 1:
                    if (i >= n || j >= m || bases_match(text[i], pattern[j])) return -1;
                    ++i, ++j, ++edits;
                    break;
                case 2:
                    if (j >= m) return -1;
                    ++j, ++edits;
                    break;
                default:
                    if (i >= n) return -1;
                    ++i, ++edits;
                    break;
            }
        }
    }
    return i == n && j == m ? edits : -1;
}

typedef struct {
    int64_t lo, hi, bad;
    const uint8_t *text, *pattern, *runs;
    const int64_t *text_off, *text_len, *pat_off, *pat_len, *cigar_off, *distance;
} replay_job;

static void* replay_worker(void* arg) {
    replay_job* j = (replay_job*)arg;
    for (int64_t k = j->lo; k < j->hi; ++k) {
        const int64_t e = orc_replay_runs(j->text + j->text_off[k], j->text_len[k],
                                          j->pattern + j->pat_off[k], j->pat_len[k],
                                          j->runs + j->cigar_off[k],
                                          j->cigar_off[k + 1] - j->cigar_off[k]);
        if (e < 0 || e != j->distance[k]) ++j->bad;
    }
    return NULL;
}

int64_t orc_replay_batch(int64_t n_pairs, const uint8_t* text, const int64_t* text_off,
                         const int64_t* text_len, const uint8_t* pattern, const int64_t* pat_off,
                         const int64_t* pat_len, const uint8_t* runs, const int64_t* cigar_off,
                         const int64_t* distance, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 128) threads = 128;
    pthread_t th[128];
    replay_job jobs[128];
    const int64_t chunk = (n_pairs + threads - 1) / threads;
    int started = 0;
    for (int t = 0; t < threads; ++t) {
        replay_job* j = &jobs[t];
        j->lo = t * chunk;
        j->hi = j->lo + chunk < n_pairs ? j->lo + chunk : n_pairs;
        j->bad = 0;
        j->text = text; j->pattern = pattern; j->runs = runs;
        j->text_off = text_off; j->text_len = text_len; j->pat_off = pat_off;
        j->pat_len = pat_len; j->cigar_off = cigar_off; j->distance = distance;
        if (j->lo >= j->hi) break;
        pthread_create(&th[t], NULL, replay_worker, j);
        ++started;
    }
    int64_t bad = 0;
    for (int t = 0; t < started; ++t) {
        pthread_join(th[t], NULL);
        bad += jobs[t].bad;
    }
    return bad;
}

/* ---- exact oracle of the accuracy sweep (proj/src/oracle.cpp, sweep.cpp) ---- */

/* global_align, proj/src/oracle.cpp:39-89 */
int orc_global_align(const uint8_t* text, int64_t n, const uint8_t* pattern, int64_t m,
                     orc_result* out, char* err, size_t errlen) {
    memset(out, 0, sizeof *out);
    if (n > 100000 || m > 100000)
        return fail(err, errlen, ORC_INPUT,
                    "global_align: sequence longer than the 10^5 quadratic-cost guard");
    if ((n + 1) * (m + 1) > ((int64_t)1 << 30))
        return fail(err, errlen, ORC_INPUT,
                    "global_align: pair too large for the exact traceback matrix");
    uint8_t* move = (uint8_t*)malloc((size_t)((n + 1) * (m + 1)));
    int* prev = (int*)malloc(sizeof(int) * (size_t)(m + 1));
    int* cur = (int*)malloc(sizeof(int) * (size_t)(m + 1));
    if (!move || !prev || !cur) {
        free(move), free(prev), free(cur);
        return fail(err, errlen, ORC_INTERNAL, "out of memory");
    }
#define AT(i, j) ((size_t)(i) * (size_t)(m + 1) + (size_t)(j))
    for (int64_t j = 0; j <= m; ++j) {
        prev[j] = (int)j;
        move[AT(0, j)] = 3;
    }
    for (int64_t i = 1; i <= n; ++i) {
        cur[0] = (int)i;
        move[AT(i, 0)] = 2;
        for (int64_t j = 1; j <= m; ++j) {
            const int eq = text[i - 1] == pattern[j - 1] && text[i - 1] < 4;
            int best = prev[j - 1] + (eq ? 0 : 1);
            uint8_t mv = eq ? 0 : 1;
            if (prev[j] + 1 < best) best = prev[j] + 1, mv = 2;
            if (cur[j - 1] + 1 < best) best = cur[j - 1] + 1, mv = 3;
            cur[j] = best;
            move[AT(i, j)] = mv;
        }
        int* t = prev;
        prev = cur;
        cur = t;
    }
    out->distance = prev[m];
    /* backward walk, then the runs re-appended in forward order */
    cigar_t rev = {0};
    int64_t i = n, j = m;
    while (i > 0 || j > 0) {
        switch (move[AT(i, j)]) {
            case 0: cigar_append(&rev, '=', 1), --i, --j; break;
            case 1: cigar_append(&rev, 'X', 1), --i, --j; break;
            case 2: cigar_append(&rev, 'D', 1), --i; break;
            default: cigar_append(&rev, 'I', 1), --j; break;
        }
    }
#undef AT
    free(move), free(prev), free(cur);
    cigar_t c = {0};
    for (int64_t k = rev.n - 1; k >= 0; --k) cigar_append(&c, rev.ops[k], rev.lens[k]);
    free(rev.ops), free(rev.lens);
    out->found = 1;
    out->windows = 1;
    return finish(out, &c, ORC_OK);
}

/* score_cigar, proj/src/oracle.cpp:91-115 */
int64_t orc_score_cigar(const orc_result* r, int match_bonus, int mismatch_penalty, int gap_open,
                        int gap_extend) {
    int64_t score = 0;
    char prev_op = 0;
    for (int64_t k = 0; k < r->n_runs; ++k) {
        const char op = r->ops[k];
        const int64_t len = r->lens[k];
        if (op == '=') score += (int64_t)match_bonus * len;
        else if (op == 'X') score -= (int64_t)mismatch_penalty * len;
        else if (op == prev_op) score -= (int64_t)gap_extend * len;
        else score -= gap_open + (int64_t)gap_extend * len;
        prev_op = op;
    }
    return score;
}

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : x > y;
}

/* worst_quantile, proj/src/sweep.cpp:11-19 */
int64_t orc_worst_quantile(int64_t* scores, int64_t n, double p) {
    qsort(scores, (size_t)n, sizeof *scores, cmp_i64);
    int64_t rank = (int64_t)ceil(p * (double)n);
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    return scores[rank - 1];
}

/* ---- whole-config digests (tests/golden/make_digests.py, ref_tool.cpp:digest_line) ---- */

#define FNV_OFF 1469598103934665603ull
#define FNV_PRIME 1099511628211ull

static uint64_t fnv_bytes(uint64_t h, const char* s, size_t len) {
    for (size_t k = 0; k < len; ++k) h = (h ^ (unsigned char)s[k]) * FNV_PRIME;
    return h;
}

typedef struct digest_job {
    int64_t b_lo, b_hi, n_pairs, block;
    const int64_t* distance;
    const int32_t* windows;
    const uint8_t* found;
    const int64_t* cigar_off;
    const uint8_t* runs;
    const uint64_t* counters;
    uint64_t* digests;
} digest_job;

/* fnv1a64 of cigar_to_string (cigar.cpp:18-25) of one pair's run bytes and its run count. */
static uint64_t cigar_hash(const uint8_t* r, int64_t nbytes, int64_t* n_runs) {
    static const char opc[4] = {'=', 'X', 'I', 'D'};
    uint64_t h = FNV_OFF;
    int64_t runs = 0;
    char num[32];
    for (int64_t k = 0; k < nbytes;) {
        const int op = r[k] >> 6;
        int64_t len = 0;
        while (k < nbytes && (r[k] >> 6) == op) len += (r[k++] & 63) + 1;
        const int w = snprintf(num, sizeof num, "%lld%c", (long long)len, opc[op]);
        h = fnv_bytes(h, num, (size_t)w);
        ++runs;
    }
    *n_runs = runs;
    return h;
}

static void* digest_worker(void* arg) {
    digest_job* j = (digest_job*)arg;
    char line[512];
    for (int64_t b = j->b_lo; b < j->b_hi; ++b) {
        const int64_t lo = b * j->block;
        const int64_t hi = lo + j->block < j->n_pairs ? lo + j->block : j->n_pairs;
        uint64_t h = FNV_OFF;
        for (int64_t k = lo; k < hi; ++k) {
            int64_t n_runs = 0;
            uint64_t ch;
            if (j->found && !j->found[k]) {
                ch = fnv_bytes(FNV_OFF, "*", 1);
            } else {
                ch = cigar_hash(j->runs + j->cigar_off[k], j->cigar_off[k + 1] - j->cigar_off[k],
                                &n_runs);
            }
            const uint64_t* c = j->counters + 7 * k;
            const int w = snprintf(line, sizeof line,
                                   "%lld\t%016llx\t%lld\t%d\t%llu\t%llu\t%llu\t%llu\t%llu\t%llu\t%llu\n",
                                   (long long)j->distance[k], (unsigned long long)ch,
                                   (long long)n_runs, (int)j->windows[k], (unsigned long long)c[0],
                                   (unsigned long long)c[1], (unsigned long long)c[2],
                                   (unsigned long long)c[3], (unsigned long long)c[4],
                                   (unsigned long long)c[5], (unsigned long long)c[6]);
            h = fnv_bytes(h, line, (size_t)w);
        }
        j->digests[b] = h;
    }
    return NULL;
}

uint64_t orc_digest_blocks(int64_t n_pairs, const int64_t* distance, const int32_t* windows,
                           const uint8_t* found, const int64_t* cigar_off, const uint8_t* runs,
                           const uint64_t* counters, int64_t block, uint64_t* digests,
                           int threads) {
    if (block < 1) block = 1;
    if (threads < 1) threads = 1;
    if (threads > 128) threads = 128;
    const int64_t n_blocks = (n_pairs + block - 1) / block;
    pthread_t th[128];
    digest_job jobs[128];
    const int64_t per = (n_blocks + threads - 1) / threads;
    int started = 0;
    for (int t = 0; t < threads; ++t) {
        digest_job* j = &jobs[t];
        j->b_lo = t * per;
        j->b_hi = j->b_lo + per < n_blocks ? j->b_lo + per : n_blocks;
        if (j->b_lo >= j->b_hi) break;
        j->n_pairs = n_pairs; j->block = block; j->distance = distance; j->windows = windows;
        j->found = found; j->cigar_off = cigar_off; j->runs = runs; j->counters = counters;
        j->digests = digests;
        pthread_create(&th[t], NULL, digest_worker, j);
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    uint64_t total = FNV_OFF;
    char hex[32];
    for (int64_t b = 0; b < n_blocks; ++b) {
        snprintf(hex, sizeof hex, "%016llx", (unsigned long long)digests[b]);
        total = fnv_bytes(total, hex, 16);
    }
    return total;
}
