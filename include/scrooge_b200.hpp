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

}  // namespace scrooge_b200
