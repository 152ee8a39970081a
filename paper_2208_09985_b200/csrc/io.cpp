// Pair-file readers and result writers behind the C ABI (include/scrooge_b200.h):
// the ingest and output formats around the aligner.
//
// Readers follow proj/src/io.cpp (read_pairs_tsv :66-94, read_fasta :37-64,
// read_pairs_fasta :96-112, read_pairs :114-121): same field rules, same
// error messages. Sequences are encoded to 1-byte codes while they are read
// and packed to 2 bits per base (+ N mask) by sg_pack. Writers follow
// write_batch_tsv (proj/src/batch.cpp:106-113) and the CLI's JSON
// (proj/tools/main.cpp:77-88, nlohmann::json dump(2): keys in sorted order).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/scrooge_b200.h"

namespace sgk {
int set_error_msg(int code, const std::string& msg);  // host.cu
}

namespace {

struct Codes {  // 1-byte codes of all texts / patterns, before packing
    std::vector<uint8_t> text, pattern;
    std::vector<int64_t> toff, tlen, poff, plen;
};

struct PairFileOwner {
    std::vector<std::string> ids;
    std::vector<const char*> id_ptrs;
};

inline uint8_t code_of(unsigned char c) {  // toupper then encode_base (encode.hpp)
    switch (c) {
        case 'A': case 'a': return 0;
        case 'C': case 'c': return 1;
        case 'G': case 'g': return 2;
        case 'T': case 't': return 3;
        default: return 4;
    }
}

// Whole-file line reader with std::getline semantics ('\n' separated, the
// last line may lack it) and strip_cr.
struct LineReader {
    std::FILE* f = nullptr;
    std::vector<char> buf;
    size_t pos = 0, len = 0;
    bool eof = false;
    explicit LineReader(std::FILE* fp) : f(fp), buf(size_t{1} << 22) {}
    bool next(std::string& line) {
        line.clear();
        for (;;) {
            if (pos == len) {
                if (eof) return !line.empty();
                len = std::fread(buf.data(), 1, buf.size(), f);
                pos = 0;
                if (len == 0) {
                    eof = true;
                    return !line.empty();
                }
            }
            const char* s = buf.data() + pos;
            const void* nl = std::memchr(s, '\n', len - pos);
            if (nl) {
                const size_t k = static_cast<const char*>(nl) - s;
                line.append(s, k);
                pos += k + 1;
                break;
            }
            line.append(s, len - pos);
            pos = len;
        }
        return true;
    }
};

struct File {
    std::FILE* f;
    explicit File(const std::string& path) : f(std::fopen(path.c_str(), "rb")) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

void strip_cr(std::string& s) {
    if (!s.empty() && s.back() == '\r') s.pop_back();
}

struct InputError {
    std::string msg;
};

void append_codes(std::vector<uint8_t>& dst, const char* s, size_t n) {
    const size_t b = dst.size();
    dst.resize(b + n);
    for (size_t i = 0; i < n; ++i) dst[b + i] = code_of(static_cast<unsigned char>(s[i]));
}

void check_unique_ids(const std::vector<std::string>& ids) {
    std::unordered_set<std::string> seen;
    for (const std::string& id : ids)
        if (!seen.insert(id).second) throw InputError{"duplicate pair id '" + id + "'"};
}

void read_tsv(const std::string& path, std::vector<std::string>& ids, Codes& c) {
    File fh(path);
    if (!fh.f) throw InputError{"cannot open '" + path + "'"};
    LineReader lr(fh.f);
    std::string line;
    size_t lineno = 0;
    while (lr.next(line)) {
        ++lineno;
        strip_cr(line);
        if (line.empty()) continue;
        const size_t t1 = line.find('\t');
        const size_t t2 = t1 == std::string::npos ? std::string::npos : line.find('\t', t1 + 1);
        if (t1 == std::string::npos || t2 == std::string::npos ||
            line.find('\t', t2 + 1) != std::string::npos)
            throw InputError{path + ":" + std::to_string(lineno) +
                             ": expected exactly 3 tab-separated fields"};
        if (t1 == 0) throw InputError{path + ":" + std::to_string(lineno) + ": empty pair id"};
        if (t2 == t1 + 1 || t2 + 1 == line.size())
            throw InputError{path + ":" + std::to_string(lineno) + ": empty sequence"};
        ids.emplace_back(line, 0, t1);
        c.toff.push_back(static_cast<int64_t>(c.text.size()));
        c.tlen.push_back(static_cast<int64_t>(t2 - t1 - 1));
        append_codes(c.text, line.data() + t1 + 1, t2 - t1 - 1);
        c.poff.push_back(static_cast<int64_t>(c.pattern.size()));
        c.plen.push_back(static_cast<int64_t>(line.size() - t2 - 1));
        append_codes(c.pattern, line.data() + t2 + 1, line.size() - t2 - 1);
    }
    check_unique_ids(ids);
}

// read_fasta (io.cpp:37-64) into names + concatenated codes.
void read_fasta(const std::string& path, std::vector<std::string>& names, std::vector<uint8_t>& seq,
                std::vector<int64_t>& off, std::vector<int64_t>& len) {
    File fh(path);
    if (!fh.f) throw InputError{"cannot open '" + path + "'"};
    LineReader lr(fh.f);
    std::string line;
    size_t lineno = 0;
    while (lr.next(line)) {
        ++lineno;
        strip_cr(line);
        if (line.empty()) continue;
        if (line[0] == '>') {
            std::string name = line.substr(1, line.find_first_of(" \t", 1) - 1);
            if (name.empty())
                throw InputError{path + ":" + std::to_string(lineno) + ": unnamed FASTA record"};
            names.push_back(std::move(name));
            off.push_back(static_cast<int64_t>(seq.size()));
            len.push_back(0);
        } else {
            if (names.empty())
                throw InputError{path + ":" + std::to_string(lineno) +
                                 ": sequence data before the first '>' header"};
            append_codes(seq, line.data(), line.size());
            len.back() += static_cast<int64_t>(line.size());
        }
    }
    for (size_t k = 0; k < names.size(); ++k)
        if (len[k] == 0) throw InputError{path + ": record '" + names[k] + "' has no sequence"};
}

void read_fasta_pairs(const std::string& input, std::vector<std::string>& ids, Codes& c) {
    const size_t comma = input.find(',');
    if (comma == std::string::npos)
        throw InputError{"fasta-pair input must name two files as '<text.fa>,<pattern.fa>'"};
    std::vector<std::string> tnames, pnames;
    read_fasta(input.substr(0, comma), tnames, c.text, c.toff, c.tlen);
    read_fasta(input.substr(comma + 1), pnames, c.pattern, c.poff, c.plen);
    if (tnames.size() != pnames.size())
        throw InputError{"FASTA pair files hold " + std::to_string(tnames.size()) + " and " +
                         std::to_string(pnames.size()) + " records; counts must match"};
    ids = std::move(tnames);
    check_unique_ids(ids);
}

// nlohmann::json string escaping (dump, ensure_ascii = false)
void json_string(std::string& out, const char* s) {
    out += '"';
    for (const unsigned char* p = reinterpret_cast<const unsigned char*>(s); *p; ++p) {
        switch (*p) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (*p < 0x20) {
                    char u[8];
                    std::snprintf(u, sizeof u, "\\u%04x", *p);
                    out += u;
                } else {
                    out += static_cast<char>(*p);
                }
        }
    }
    out += '"';
}

}  // namespace

extern "C" {

int sg_read_pairs(const char* input, int format, sg_pair_file* out) {
    if (!out || !input) return sgk::set_error_msg(SG_INPUT, "null argument");
    std::memset(out, 0, sizeof *out);
    auto own = std::make_unique<PairFileOwner>();
    Codes c;
    try {
        if (format == SG_FORMAT_TSV)
            read_tsv(input, own->ids, c);
        else if (format == SG_FORMAT_FASTA_PAIR)
            read_fasta_pairs(input, own->ids, c);
        else
            return sgk::set_error_msg(SG_INPUT, "unknown input format (expected tsv or fasta-pair)");
    } catch (const InputError& e) {
        return sgk::set_error_msg(SG_INPUT, e.msg);
    } catch (const std::bad_alloc&) {
        return sgk::set_error_msg(SG_INTERNAL, "out of host memory reading '" + std::string(input) + "'");
    }
    const int64_t n = static_cast<int64_t>(own->ids.size());
    sg_pairs pv{n, c.text.data(), c.toff.data(), c.tlen.data(), c.pattern.data(), c.poff.data(),
                c.plen.data()};
    const int rc = sg_pack(&pv, &out->packed);
    if (rc) return rc;
    own->id_ptrs.resize(own->ids.size());
    for (size_t k = 0; k < own->ids.size(); ++k) own->id_ptrs[k] = own->ids[k].c_str();
    out->n_pairs = n;
    out->ids = own->id_ptrs.data();
    out->_owner = own.release();
    return SG_OK;
}

void sg_pair_file_free(sg_pair_file* f) {
    if (!f) return;
    sg_packed_free(&f->packed);
    delete static_cast<PairFileOwner*>(f->_owner);
    std::memset(f, 0, sizeof *f);
}

int sg_write_results(const char* path, const sg_pair_file* pairs, const sg_results* res, int json) {
    if (!pairs || !res || res->n_pairs != pairs->n_pairs)
        return sgk::set_error_msg(SG_INPUT, "results do not match the pair file");
    std::FILE* f = stdout;
    const bool to_file = path && std::strcmp(path, "-") != 0 && path[0];
    if (to_file && !(f = std::fopen(path, "wb")))  // OutputTarget::open, main.cpp:27-32
        return sgk::set_error_msg(SG_INPUT, "cannot write '" + std::string(path) + "'");
    std::string out, cig;
    static const char kOp[4] = {'=', 'X', 'I', 'D'};
    auto cigar = [&](int64_t k) -> const std::string& {  // cigar_to_string, cigar.cpp:18-25
        cig.clear();
        if (!res->found[k]) {
            cig = "*";
            return cig;
        }
        int op = -1;
        long long len = 0;
        for (int64_t b = res->cigar_off[k]; b < res->cigar_off[k + 1]; ++b) {
            const int o = res->runs[b] >> 6;
            if (o != op && op >= 0) {
                cig += std::to_string(len);
                cig += kOp[op];
                len = 0;
            }
            op = o;
            len += (res->runs[b] & 63) + 1;
        }
        if (op >= 0) {
            cig += std::to_string(len);
            cig += kOp[op];
        }
        return cig;
    };
    const int64_t n = res->n_pairs;
    if (json) {
        out = n ? "[\n" : "[]";
        for (int64_t k = 0; k < n; ++k) {
            out += "  {\n    \"cigar\": ";
            json_string(out, cigar(k).c_str());
            out += ",\n    \"distance\": " + std::to_string(res->distance[k]);
            out += ",\n    \"id\": ";
            json_string(out, pairs->ids[k]);
            out += ",\n    \"windows\": " + std::to_string(res->windows[k]) + "\n  }";
            out += k + 1 < n ? ",\n" : "\n]";
            if (out.size() > (size_t{1} << 24)) {
                std::fwrite(out.data(), 1, out.size(), f);
                out.clear();
            }
        }
        out += "\n";
    } else {
        for (int64_t k = 0; k < n; ++k) {
            out += pairs->ids[k];
            out += '\t';
            out += std::to_string(res->distance[k]);
            out += '\t';
            out += cigar(k);
            out += '\n';
            if (out.size() > (size_t{1} << 24)) {
                std::fwrite(out.data(), 1, out.size(), f);
                out.clear();
            }
        }
    }
    std::fwrite(out.data(), 1, out.size(), f);
    const bool ok = std::ferror(f) == 0;
    if (to_file) std::fclose(f);
    else std::fflush(f);
    if (!ok) return sgk::set_error_msg(SG_INPUT, "cannot write '" + std::string(to_file ? path : "-") + "'");
    return SG_OK;
}

}  // extern "C"
