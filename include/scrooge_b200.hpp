// scrooge_b200.hpp — header-only C++ drop-in for the reference aligner API
// (/root/reference/proj/include/scrooge/{aligner,batch,cigar,errors}.hpp),
// implemented over the C ABI in scrooge_b200.h (link libscrooge_b200.so).
//
// Same names, argument meaning and error behaviour as the reference:
//   scrooge_b200::AlignerConfig      <- scrooge::AlignerConfig      (aligner.hpp:12-31)
//   scrooge_b200::align              <- scrooge::align              (aligner.hpp:45)
//   scrooge_b200::run_batch          <- scrooge::run_batch          (batch.hpp:33-34)
//   scrooge_b200::write_batch_tsv    <- scrooge::write_batch_tsv    (batch.hpp:37-38)
//   scrooge_b200::cigar_to_string    <- scrooge::cigar_to_string    (cigar.hpp:26)
//   InputError / ConfigError / InternalError / OutOfStoredRegionError (errors.hpp:10-34)
// A caller switches by replacing `scrooge::` with `scrooge_b200::`. The
// Workspace argument of align() is accepted and ignored (device buffers are
// owned by the library); run_batch's `threads` keeps its validation.
#pragma once

#include <cstdint>
#include <ostream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "scrooge_b200.h"

namespace scrooge_b200 {

class InputError : public std::runtime_error {
public:
    explicit InputError(const std::string& w) : std::runtime_error(w) {}
};
class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
class InternalError : public std::logic_error {
public:
    explicit InternalError(const std::string& w) : std::logic_error(w) {}
};
class OutOfStoredRegionError : public InternalError {
public:
    explicit OutOfStoredRegionError(const std::string& w) : InternalError(w) {}
};
class DeviceError : public std::runtime_error {  // no reference equivalent
public:
    explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

[[noreturn]] inline void throw_status(int rc, std::string msg) {
    switch (rc) {
        case SG_INPUT: throw InputError(msg);
        case SG_CONFIG: throw ConfigError(msg);
        case SG_INTERNAL: throw InternalError(msg);
        default: throw DeviceError(msg);
    }
}

inline void check(int rc) {
    if (rc != SG_OK) throw_status(rc, sg_last_error());
}

using BaseCode = std::uint8_t;
struct CodeView {  // std::span<const BaseCode> stand-in (C++17)
    const BaseCode* data_ = nullptr;
    std::size_t size_ = 0;
    CodeView() = default;
    CodeView(const BaseCode* d, std::size_t n) : data_(d), size_(n) {}
    CodeView(const std::vector<BaseCode>& v) : data_(v.data()), size_(v.size()) {}
    const BaseCode* data() const { return data_; }
    std::size_t size() const { return size_; }
    bool empty() const { return size_ == 0; }
};

inline BaseCode encode_base(char c) {
    switch (c) {
        case 'A': case 'a': return 0;
        case 'C': case 'c': return 1;
        case 'G': case 'g': return 2;
        case 'T': case 't': return 3;
        default: return 4;
    }
}

inline std::vector<BaseCode> encode_sequence(std::string_view s) {
    std::vector<BaseCode> out(s.size());
    for (std::size_t i = 0; i < s.size(); ++i) out[i] = encode_base(s[i]);
    return out;
}

struct CigarOp {
    char op = '=';
    std::int64_t len = 0;
    bool operator==(const CigarOp& o) const { return op == o.op && len == o.len; }
};
using Cigar = std::vector<CigarOp>;

inline std::string cigar_to_string(const Cigar& cigar) {
    std::string s;
    for (const CigarOp& r : cigar) {
        s += std::to_string(r.len);
        s += r.op;
    }
    return s;
}

struct InstrumentationCounters {
    std::uint64_t stored_bits = 0, table_writes = 0, table_reads = 0, rows_computed = 0,
                  cells_computed = 0, rows_possible = 0, baseline_equiv_bits = 0;
    void add(const InstrumentationCounters& o) {
        stored_bits += o.stored_bits;
        table_writes += o.table_writes;
        table_reads += o.table_reads;
        rows_computed += o.rows_computed;
        cells_computed += o.cells_computed;
        rows_possible += o.rows_possible;
        baseline_equiv_bits += o.baseline_equiv_bits;
    }
};

struct AlignerConfig {
    int W = 64;
    int O = 33;
    bool sene = true;
    bool dent = true;
    bool early_termination = true;
    enum class Mode { Windowed, SingleWindow };
    Mode mode = Mode::Windowed;
    int k_single = 1024;

    sg_config c() const {
        sg_config r;
        r.W = W;
        r.O = O;
        r.sene = sene;
        r.dent = dent;
        r.early_termination = early_termination;
        r.single_window = mode == Mode::SingleWindow;
        r.k_single = k_single;
        return r;
    }
    void validate() const {
        const sg_config cc = c();
        check(sg_validate_config(&cc));
    }
};

struct AlignmentResult {
    std::int64_t distance = 0;
    Cigar cigar;
    int windows = 0;
    InstrumentationCounters counters;
};

struct Workspace {};  // device state is owned by the library

struct SeqPairRecord {
    std::string id;
    std::string text;
    std::string pattern;
};

struct PairOutcome {
    bool found = true;
    std::int64_t distance = -1;
    Cigar cigar;
    int windows = 0;
    InstrumentationCounters counters;
};

struct BatchResult {
    std::vector<PairOutcome> outcomes;
    InstrumentationCounters total;
    double align_seconds = 0.0;
    double pairs_per_second = 0.0;
};

namespace detail {

struct Results {
    sg_results r{};
    ~Results() { sg_results_free(&r); }
};

inline InstrumentationCounters counters_of(const sg_results& r, std::int64_t k) {
    const std::uint64_t* c = r.counters + k * SG_CNT_COUNT;
    InstrumentationCounters o;
    o.stored_bits = c[0];
    o.table_writes = c[1];
    o.table_reads = c[2];
    o.rows_computed = c[3];
    o.cells_computed = c[4];
    o.rows_possible = c[5];
    o.baseline_equiv_bits = c[6];
    return o;
}

inline Cigar cigar_of(const sg_results& r, std::int64_t k) {
    static const char kOp[4] = {'=', 'X', 'I', 'D'};
    Cigar out;
    for (std::int64_t b = r.cigar_off[k]; b < r.cigar_off[k + 1]; ++b) {
        const int op = r.runs[b] >> 6;
        const std::int64_t len = (r.runs[b] & 63) + 1;
        if (!out.empty() && out.back().op == kOp[op])
            out.back().len += len;
        else
            out.push_back({kOp[op], len});
    }
    return out;
}

// Replaces "pair '<index>'" in a library message by the caller's pair id.
inline std::string with_id(const std::string& msg, const std::vector<SeqPairRecord>& pairs) {
    const std::string key = "pair '";
    if (msg.compare(0, key.size(), key) != 0) return msg;
    const std::size_t end = msg.find('\'', key.size());
    if (end == std::string::npos) return msg;
    const std::size_t idx = std::stoull(msg.substr(key.size(), end - key.size()));
    if (idx >= pairs.size()) return msg;
    return key + pairs[idx].id + msg.substr(end);
}

}  // namespace detail

// align (aligner.cpp:28-85): one pair through the GPU path.
inline AlignmentResult align(CodeView text, CodeView pattern, const AlignerConfig& config) {
    config.validate();
    if (config.mode != AlignerConfig::Mode::Windowed)
        throw ConfigError("align() requires windowed mode");
    if (text.empty() || pattern.empty()) throw InputError("align: empty input sequence");
    const std::int64_t zero = 0, n = static_cast<std::int64_t>(text.size()),
                       m = static_cast<std::int64_t>(pattern.size());
    sg_pairs p{1, text.data(), &zero, &n, pattern.data(), &zero, &m};
    const sg_config cc = config.c();
    detail::Results res;
    check(sg_align_batch(&cc, &p, nullptr, 0, &res.r));
    AlignmentResult out;
    out.distance = res.r.distance[0];
    out.cigar = detail::cigar_of(res.r, 0);
    out.windows = res.r.windows[0];
    out.counters = detail::counters_of(res.r, 0);
    return out;
}

inline AlignmentResult align(CodeView text, CodeView pattern, const AlignerConfig& config,
                             Workspace&) {
    return align(text, pattern, config);
}

// run_batch (batch.cpp:13-104) on `devices` (empty = device 0).
inline BatchResult run_batch(const std::vector<SeqPairRecord>& pairs, const AlignerConfig& config,
                             int threads, const std::vector<int>& devices = {}) {
    config.validate();
    if (threads < 1) throw ConfigError("thread count must be at least 1");
    const std::size_t n = pairs.size();
    std::vector<std::int64_t> toff(n), tlen(n), poff(n), plen(n);
    std::vector<BaseCode> text, pattern;
    for (std::size_t k = 0; k < n; ++k) {
        if (pairs[k].text.empty() || pairs[k].pattern.empty())
            throw InputError("pair '" + pairs[k].id + "': empty sequence");
        toff[k] = static_cast<std::int64_t>(text.size());
        tlen[k] = static_cast<std::int64_t>(pairs[k].text.size());
        poff[k] = static_cast<std::int64_t>(pattern.size());
        plen[k] = static_cast<std::int64_t>(pairs[k].pattern.size());
        for (char c : pairs[k].text) text.push_back(encode_base(c));
        for (char c : pairs[k].pattern) pattern.push_back(encode_base(c));
    }
    sg_pairs p{static_cast<std::int64_t>(n), text.data(), toff.data(), tlen.data(),
               pattern.data(), poff.data(), plen.data()};
    const sg_config cc = config.c();
    detail::Results res;
    const int rc = sg_align_batch(&cc, &p, devices.empty() ? nullptr : devices.data(),
                                  static_cast<int>(devices.size()), &res.r);
    if (rc != SG_OK) throw_status(rc, detail::with_id(sg_last_error(), pairs));
    BatchResult out;
    out.outcomes.resize(n);
    for (std::size_t k = 0; k < n; ++k) {
        PairOutcome& po = out.outcomes[k];
        po.found = res.r.found[k] != 0;
        po.distance = res.r.distance[k];
        po.cigar = detail::cigar_of(res.r, static_cast<std::int64_t>(k));
        po.windows = res.r.windows[k];
        po.counters = detail::counters_of(res.r, static_cast<std::int64_t>(k));
        out.total.add(po.counters);
    }
    out.align_seconds = res.r.align_seconds;
    out.pairs_per_second = out.align_seconds > 0 ? static_cast<double>(n) / out.align_seconds : 0;
    return out;
}

// write_batch_tsv (batch.cpp:106-113).
inline void write_batch_tsv(std::ostream& os, const std::vector<SeqPairRecord>& pairs,
                            const BatchResult& result) {
    for (std::size_t i = 0; i < pairs.size(); ++i) {
        const PairOutcome& po = result.outcomes[i];
        os << pairs[i].id << '\t' << po.distance << '\t'
           << (po.found ? cigar_to_string(po.cigar) : "*") << '\n';
    }
}

// ---- exact oracle and accuracy sweep (oracle.hpp, sweep.hpp) on the GPU

namespace oracle {

struct ScoringParams {  // oracle.hpp:14-19
    int match_bonus = 2;
    int mismatch_penalty = 4;
    int gap_open = 4;
    int gap_extend = 2;
};

struct GlobalAlignment {  // oracle.hpp:29-32
    int distance = 0;
    Cigar cigar;
};

// global_align (oracle.cpp:39-89): optimal unit-cost alignment, the reference's
// tie-breaking, computed by K7.
inline GlobalAlignment global_align(CodeView text, CodeView pattern) {
    const std::int64_t zero = 0, n = static_cast<std::int64_t>(text.size()),
                       m = static_cast<std::int64_t>(pattern.size());
    sg_pairs p{1, text.data(), &zero, &n, pattern.data(), &zero, &m};
    sg_packed_pairs packed{};
    check(sg_pack(&p, &packed));
    detail::Results res;
    const int rc = sg_global_align(&packed, 0, &res.r);
    sg_packed_free(&packed);
    check(rc);
    GlobalAlignment out;
    out.distance = static_cast<int>(res.r.distance[0]);
    out.cigar = detail::cigar_of(res.r, 0);
    return out;
}

// score_cigar (oracle.cpp:91-115).
inline std::int64_t score_cigar(const Cigar& cigar, const ScoringParams& params) {
    std::int64_t score = 0;
    char prev_op = '\0';
    for (const CigarOp& run : cigar) {
        if (run.op != '=' && run.op != 'X' && run.op != 'I' && run.op != 'D')
            throw InputError(std::string("score_cigar: unknown op '") + run.op + "'");
        if (run.len <= 0) throw InputError("score_cigar: non-positive run length");
        if (run.op == '=') score += std::int64_t{params.match_bonus} * run.len;
        else if (run.op == 'X') score -= std::int64_t{params.mismatch_penalty} * run.len;
        else if (run.op == prev_op) score -= std::int64_t{params.gap_extend} * run.len;
        else score -= params.gap_open + std::int64_t{params.gap_extend} * run.len;
        prev_op = run.op;
    }
    return score;
}

}  // namespace oracle

struct ImprovementCombo {  // sweep.hpp:12-16
    bool sene = false;
    bool dent = false;
    bool et = false;
};

struct OverlapRule {  // sweep.hpp:19-24
    enum class Kind { HalfPlusOne, Fixed } kind = Kind::HalfPlusOne;
    int fixed = 0;
    int overlap_for(int W) const { return kind == Kind::HalfPlusOne ? W / 2 + 1 : fixed; }
};

struct SweepOptions {  // sweep.hpp:26-36
    std::vector<int> W_list;
    OverlapRule o_rule;
    std::vector<ImprovementCombo> combos;
    oracle::ScoringParams scoring;
    int threads = 1;
    bool measure_time = true;
    std::vector<int> devices;  // GPU devices (empty = device 0); no reference equivalent
};

using SweepRow = sg_sweep_row;  // sweep.hpp:38-49 (same fields)

struct SweepReport {
    std::vector<SweepRow> rows;
};

// worst_quantile (sweep.cpp:11-19).
inline std::int64_t worst_quantile(std::vector<std::int64_t> scores, double p) {
    std::int64_t out = 0;
    check(sg_worst_quantile(scores.data(), static_cast<std::int64_t>(scores.size()), p, &out));
    return out;
}

// run_sweep (sweep.cpp:40-107): the GPU aligner and the GPU exact oracle.
inline SweepReport run_sweep(const std::vector<SeqPairRecord>& pairs, const SweepOptions& options) {
    const std::size_t n = pairs.size();
    std::vector<std::int64_t> toff(n), tlen(n), poff(n), plen(n);
    std::vector<BaseCode> text, pattern;
    for (std::size_t k = 0; k < n; ++k) {
        toff[k] = static_cast<std::int64_t>(text.size());
        tlen[k] = static_cast<std::int64_t>(pairs[k].text.size());
        poff[k] = static_cast<std::int64_t>(pattern.size());
        plen[k] = static_cast<std::int64_t>(pairs[k].pattern.size());
        for (char c : pairs[k].text) text.push_back(encode_base(c));
        for (char c : pairs[k].pattern) pattern.push_back(encode_base(c));
    }
    sg_pairs p{static_cast<std::int64_t>(n), text.data(), toff.data(), tlen.data(),
               pattern.data(), poff.data(), plen.data()};
    sg_packed_pairs packed{};
    if (n) check(sg_pack(&p, &packed));
    std::vector<std::uint8_t> combos;
    for (const ImprovementCombo& c : options.combos)
        combos.push_back(static_cast<std::uint8_t>((c.sene ? 1 : 0) | (c.dent ? 2 : 0) | (c.et ? 4 : 0)));
    sg_sweep_options o{};
    o.W_list = options.W_list.data();
    o.n_W = static_cast<std::int32_t>(options.W_list.size());
    o.o_fixed = options.o_rule.kind == OverlapRule::Kind::HalfPlusOne ? -1 : options.o_rule.fixed;
    o.combos = combos.data();
    o.n_combos = static_cast<std::int32_t>(combos.size());
    o.scoring = {options.scoring.match_bonus, options.scoring.mismatch_penalty,
                 options.scoring.gap_open, options.scoring.gap_extend};
    o.measure_time = options.measure_time ? 1 : 0;
    SweepReport report;
    report.rows.resize(options.W_list.size() * combos.size());
    const int rc = sg_sweep(&o, n ? &packed : nullptr,
                            options.devices.empty() ? nullptr : options.devices.data(),
                            static_cast<int>(options.devices.size()), report.rows.data());
    if (n) sg_packed_free(&packed);
    check(rc);
    return report;
}

// sweep_csv (sweep.cpp:110-127).
inline std::string sweep_csv(const SweepReport& report) {
    const std::int64_t nr = static_cast<std::int64_t>(report.rows.size());
    const std::int64_t len = sg_sweep_format(report.rows.data(), nr, 0, nullptr, 0);
    std::string s(static_cast<std::size_t>(len) + 1, '\0');
    sg_sweep_format(report.rows.data(), nr, 0, &s[0], len + 1);
    s.resize(static_cast<std::size_t>(len));
    return s;
}

}  // namespace scrooge_b200
