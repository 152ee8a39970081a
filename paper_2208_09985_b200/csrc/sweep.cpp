// The accuracy sweep (run_sweep, proj/src/sweep.cpp:40-107) over the C ABI:
// the GPU aligner for every (W, combo) and the GPU exact oracle (K7,
// sg_global_align) in place of the quadratic CPU global_align. Scoring,
// quantiles and the report formats follow the reference exactly
// (score_cigar proj/src/oracle.cpp:91-115; worst_quantile sweep.cpp:11-19;
// sweep_csv sweep.cpp:110-127; the CLI's JSON proj/tools/main.cpp:90-111).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/scrooge_b200.h"

namespace sgk {
int set_error_msg(int code, const std::string& msg);  // host.cu
}

namespace {

struct Quantiles {
    int64_t q500, q100, q010, q001;
};

int64_t worst_quantile(std::vector<int64_t> scores, double p) {  // non-empty, p in (0, 1]
    std::sort(scores.begin(), scores.end());  // ascending = worst first
    const size_t n = scores.size();
    size_t rank = static_cast<size_t>(std::ceil(p * static_cast<double>(n)));
    rank = std::min(std::max<size_t>(rank, 1), n);
    return scores[rank - 1];
}

Quantiles quantiles(const std::vector<int64_t>& s) {
    return {worst_quantile(s, 0.5), worst_quantile(s, 0.1), worst_quantile(s, 0.01),
            worst_quantile(s, 0.001)};
}

std::string fmt6(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.6f", v);
    return buf;
}

// nlohmann::json's number output: the shortest round-trip digits, printed as
// an integer with ".0", a plain decimal, or d.ddde+XX.
std::string json_double(double v) {
    if (v == 0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    int prec = 1;
    for (; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s = buf;  // [-]d.ddde[+-]XX
    const bool neg = s[0] == '-';
    if (neg) s.erase(0, 1);
    const size_t e = s.find('e');
    std::string digits = s.substr(0, 1) + (e > 2 ? s.substr(2, e - 2) : "");
    const int exp10 = std::atoi(s.c_str() + e + 1);
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // value = 0.digits * 10^n
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
    } else if (-5 < n && n <= 0) {
        out = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", n - 1 < 0 ? '-' : '+', std::abs(n - 1));
        out += eb;
    }
    return neg ? "-" + out : out;
}

int fail(int code, const std::string& msg) { return sgk::set_error_msg(code, msg); }

}  // namespace

extern "C" {

void sg_scoring_default(sg_scoring* s) {
    s->match_bonus = 2;
    s->mismatch_penalty = 4;
    s->gap_open = 4;
    s->gap_extend = 2;
}

int64_t sg_score_cigar(const sg_results* res, int64_t k, const sg_scoring* sp) {
    static const char kOps[4] = {'=', 'X', 'I', 'D'};
    int64_t score = 0;
    char prev_op = '\0';
    const uint8_t* b = res->runs + res->cigar_off[k];
    const uint8_t* e = res->runs + res->cigar_off[k + 1];
    while (b < e) {  // merged runs, as cigar_append builds them
        const char op = kOps[*b >> 6];
        int64_t len = 0;
        while (b < e && kOps[*b >> 6] == op) len += (*b++ & 63) + 1;
        switch (op) {
            case '=': score += int64_t{sp->match_bonus} * len; break;
            case 'X': score -= int64_t{sp->mismatch_penalty} * len; break;
            default:  // each maximal I or D run is one gap
                if (op == prev_op)
                    score -= int64_t{sp->gap_extend} * len;
                else
                    score -= sp->gap_open + int64_t{sp->gap_extend} * len;
                break;
        }
        prev_op = op;
    }
    return score;
}

int sg_worst_quantile(const int64_t* scores, int64_t n, double p, int64_t* out) {
    if (n <= 0) return fail(SG_INPUT, "quantile of an empty score list");
    if (!(p > 0.0 && p <= 1.0)) return fail(SG_INPUT, "quantile fraction must lie in (0, 1]");
    *out = worst_quantile(std::vector<int64_t>(scores, scores + n), p);
    return SG_OK;
}

int sg_sweep(const sg_sweep_options* opt, const sg_packed_pairs* pairs, const int* devices,
             int n_devices, sg_sweep_row* rows) {
    if (!pairs || pairs->n_pairs <= 0) return fail(SG_INPUT, "sweep: empty dataset");
    if (opt->n_W <= 0) return fail(SG_INPUT, "sweep: empty W list");
    if (opt->n_combos <= 0) return fail(SG_INPUT, "sweep: no improvement combinations");
    const int64_t n = pairs->n_pairs;

    // oracle baseline, once per pair (K7)
    sg_results ex;
    int rc = sg_global_align(pairs, devices && n_devices > 0 ? devices[0] : 0, &ex);
    if (rc) return rc;
    std::vector<int64_t> oracle_dist(static_cast<size_t>(n)), oracle_scores(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
        oracle_dist[static_cast<size_t>(k)] = ex.distance[k];
        oracle_scores[static_cast<size_t>(k)] = sg_score_cigar(&ex, k, &opt->scoring);
    }
    sg_results_free(&ex);
    const Quantiles oq = quantiles(oracle_scores);

    size_t r = 0;
    std::vector<int64_t> scores(static_cast<size_t>(n));
    for (int w = 0; w < opt->n_W; ++w) {
        const int W = opt->W_list[w];
        const int O = opt->o_fixed < 0 ? W / 2 + 1 : opt->o_fixed;
        for (int c = 0; c < opt->n_combos; ++c) {
            sg_config cfg;
            sg_config_default(&cfg);
            cfg.W = W;
            cfg.O = O;
            cfg.sene = opt->combos[c] & 1;
            cfg.dent = (opt->combos[c] >> 1) & 1;
            cfg.early_termination = (opt->combos[c] >> 2) & 1;
            if ((rc = sg_validate_config(&cfg))) return rc;
            sg_results br;
            if ((rc = sg_align_packed(&cfg, pairs, devices, n_devices, &br))) return rc;
            int64_t optimal = 0;
            for (int64_t k = 0; k < n; ++k) {
                scores[static_cast<size_t>(k)] = sg_score_cigar(&br, k, &opt->scoring);
                if (br.distance[k] == oracle_dist[static_cast<size_t>(k)]) ++optimal;
            }
            const Quantiles q = quantiles(scores);
            sg_sweep_row& row = rows[r++];
            std::memset(&row, 0, sizeof row);
            row.W = W;
            row.O = O;
            row.sene = cfg.sene;
            row.dent = cfg.dent;
            row.et = cfg.early_termination;
            row.q500 = q.q500;
            row.q100 = q.q100;
            row.q010 = q.q010;
            row.q001 = q.q001;
            row.frac_optimal = static_cast<double>(optimal) / static_cast<double>(n);
            const uint64_t* t = br.total;
            row.mean_rows_frac = t[SG_CNT_ROWS_POSSIBLE] > 0
                                     ? static_cast<double>(t[SG_CNT_ROWS_COMPUTED]) /
                                           static_cast<double>(t[SG_CNT_ROWS_POSSIBLE])
                                     : 0.0;
            row.stored_bits_ratio = t[SG_CNT_STORED_BITS] > 0
                                        ? static_cast<double>(t[SG_CNT_BASELINE_EQUIV_BITS]) /
                                              static_cast<double>(t[SG_CNT_STORED_BITS])
                                        : 0.0;
            row.pairs_per_s = opt->measure_time && br.align_seconds > 0
                                  ? static_cast<double>(n) / br.align_seconds
                                  : 0.0;
            row.oracle_q500 = oq.q500;
            row.oracle_q100 = oq.q100;
            row.oracle_q010 = oq.q010;
            row.oracle_q001 = oq.q001;
            sg_results_free(&br);
        }
    }
    return SG_OK;
}

int64_t sg_sweep_format(const sg_sweep_row* rows, int64_t n_rows, int json, char* buf, int64_t cap) {
    std::string out;
    auto i64 = [](int64_t v) { return std::to_string(v); };
    if (!json) {
        out = "W,O,sene,dent,et,q500,q100,q010,q001,frac_optimal,mean_rows_frac,"
              "stored_bits_ratio,pairs_per_s,oracle_q500,oracle_q100,oracle_q010,oracle_q001\n";
        for (int64_t k = 0; k < n_rows; ++k) {
            const sg_sweep_row& r = rows[k];
            out += std::to_string(r.W) + ',' + std::to_string(r.O) + ',';
            out += std::string(r.sene ? "1" : "0") + ',' + (r.dent ? "1" : "0") + ',' +
                   (r.et ? "1" : "0") + ',';
            out += i64(r.q500) + ',' + i64(r.q100) + ',' + i64(r.q010) + ',' + i64(r.q001) + ',';
            out += fmt6(r.frac_optimal) + ',' + fmt6(r.mean_rows_frac) + ',' +
                   fmt6(r.stored_bits_ratio) + ',' + fmt6(r.pairs_per_s) + ',';
            out += i64(r.oracle_q500) + ',' + i64(r.oracle_q100) + ',' + i64(r.oracle_q010) + ',' +
                   i64(r.oracle_q001) + '\n';
        }
    } else if (n_rows == 0) {
        out = "[]";
    } else {  // json::dump(2): keys sorted
        out = "[\n";
        for (int64_t k = 0; k < n_rows; ++k) {
            const sg_sweep_row& r = rows[k];
            auto b = [](int v) { return std::string(v ? "true" : "false"); };
            const std::pair<const char*, std::string> kv[] = {
                {"O", std::to_string(r.O)},
                {"W", std::to_string(r.W)},
                {"dent", b(r.dent)},
                {"et", b(r.et)},
                {"frac_optimal", json_double(r.frac_optimal)},
                {"mean_rows_frac", json_double(r.mean_rows_frac)},
                {"oracle_q001", i64(r.oracle_q001)},
                {"oracle_q010", i64(r.oracle_q010)},
                {"oracle_q100", i64(r.oracle_q100)},
                {"oracle_q500", i64(r.oracle_q500)},
                {"pairs_per_s", json_double(r.pairs_per_s)},
                {"q001", i64(r.q001)},
                {"q010", i64(r.q010)},
                {"q100", i64(r.q100)},
                {"q500", i64(r.q500)},
                {"sene", b(r.sene)},
                {"stored_bits_ratio", json_double(r.stored_bits_ratio)},
            };
            out += "  {\n";
            for (size_t i = 0; i < sizeof kv / sizeof kv[0]; ++i) {
                out += "    \"" + std::string(kv[i].first) + "\": " + kv[i].second;
                out += i + 1 < sizeof kv / sizeof kv[0] ? ",\n" : "\n";
            }
            out += k + 1 < n_rows ? "  },\n" : "  }\n";
        }
        out += "]";
    }
    const int64_t len = static_cast<int64_t>(out.size());
    if (buf && len < cap) std::memcpy(buf, out.c_str(), static_cast<size_t>(len) + 1);
    return len;
}

}  // extern "C"
