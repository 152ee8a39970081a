// sg_align: the reference CLI's `align` / `bench` flows (proj/tools/main.cpp:
// 113-177, 287-299) on the GPU path: read pairs (TSV or FASTA pair), align on
// one or more GPUs, write TSV or JSON identical to the reference's output.
//
//   sg_align align --input pairs.tsv [--format tsv|fasta-pair] [--W 64] [--O 33]
//                  [--sene|--no-sene] [--dent|--no-dent] [--et|--no-et]
//                  [--threads N] [--output PATH] [--mode windowed|single] [--k K]
//                  [--json] [--devices 0,1,...]
//   sg_align bench ...same...   (also prints the throughput report on stderr)
//   sg_align sweep --input pairs.tsv [--format tsv|fasta-pair] [--W-list 32,64]
//                  [--O-rule half+1|fixed:N] [--combos none,sene+dent+et|all|...]
//                  [--threads N] [--report PATH] [--json] [--no-timing] [--devices 0,1,...]
//                  (the accuracy sweep, main.cpp:218-286, with the GPU exact oracle)
//
// Exit codes follow main.cpp:287-299: 1 for input/config errors ("error: ..."),
// 2 for internal errors ("internal error: ...").
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/scrooge_b200.h"

namespace {

struct CliError {
    int code;  // SG_* status
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw CliError{code, msg}; }

void check(int rc) {
    if (rc != SG_OK) fail(rc, sg_last_error());
}

int parse_int(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const long x = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end) fail(SG_INPUT, flag + ": value '" + v + "' is not an integer");
    return static_cast<int>(x);
}

struct Args {
    std::string cmd, input, format = "tsv", output, mode = "windowed";
    sg_config cfg{};
    int threads = 1;
    bool json = false;
    std::vector<int> devices;
};

Args parse(int argc, char** argv) {
    Args a;
    sg_config_default(&a.cfg);
    if (argc < 2) fail(SG_INPUT, "usage: sg_align align|bench|sweep --input FILE [options]");
    a.cmd = argv[1];
    if (a.cmd != "align" && a.cmd != "bench") fail(SG_INPUT, "unknown command '" + a.cmd + "'");
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i], v;
        const size_t eq = k.find('=');
        const bool has_eq = k.rfind("--", 0) == 0 && eq != std::string::npos;
        if (has_eq) {
            v = k.substr(eq + 1);
            k = k.substr(0, eq);
        }
        auto val = [&]() -> std::string {
            if (has_eq) return v;
            if (i + 1 >= argc) fail(SG_INPUT, k + " requires a value");
            return argv[++i];
        };
        if (k == "--input") a.input = val();
        else if (k == "--format") a.format = val();
        else if (k == "--W") a.cfg.W = parse_int(k, val());
        else if (k == "--O") a.cfg.O = parse_int(k, val());
        else if (k == "--sene") a.cfg.sene = 1;
        else if (k == "--no-sene") a.cfg.sene = 0;
        else if (k == "--dent") a.cfg.dent = 1;
        else if (k == "--no-dent") a.cfg.dent = 0;
        else if (k == "--et") a.cfg.early_termination = 1;
        else if (k == "--no-et") a.cfg.early_termination = 0;
        else if (k == "--threads") a.threads = parse_int(k, val());
        else if (k == "--output") a.output = val();
        else if (k == "--mode") a.mode = val();
        else if (k == "--k") a.cfg.k_single = parse_int(k, val());
        else if (k == "--json") a.json = true;
        else if (k == "--devices") {
            const std::string s = val();
            size_t p = 0;
            while (p <= s.size()) {
                const size_t c = s.find(',', p);
                a.devices.push_back(parse_int(k, s.substr(p, c == std::string::npos ? c : c - p)));
                if (c == std::string::npos) break;
                p = c + 1;
            }
        } else fail(SG_INPUT, "unknown option '" + k + "'");
    }
    if (a.input.empty()) fail(SG_INPUT, "--input is required");
    // finish_align_config (main.cpp:140-150)
    if (a.mode == "windowed") {
        a.cfg.single_window = 0;
    } else if (a.mode == "single") {
        a.cfg.single_window = 1;
        a.cfg.dent = 0;
    } else {
        fail(SG_INPUT, "unknown mode '" + a.mode + "' (expected windowed or single)");
    }
    return a;
}

std::vector<int> parse_list(const std::string& flag, const std::string& s) {
    std::vector<int> out;
    size_t p = 0;
    while (p <= s.size()) {
        const size_t c = s.find(',', p);
        out.push_back(parse_int(flag, s.substr(p, c == std::string::npos ? c : c - p)));
        if (c == std::string::npos) break;
        p = c + 1;
    }
    return out;
}

// Tokens as std::getline(stream, token, delim) yields them: none for an empty
// string, no trailing empty token after a final delimiter.
std::vector<std::string> getline_split(const std::string& s, char delim) {
    std::vector<std::string> out;
    size_t p = 0;
    while (p < s.size()) {
        size_t c = s.find(delim, p);
        if (c == std::string::npos) c = s.size();
        out.push_back(s.substr(p, c - p));
        p = c + 1;
    }
    return out;
}

// parse_combos, main.cpp:48-75
std::vector<uint8_t> parse_combos(const std::string& s) {
    std::vector<uint8_t> combos;
    for (const std::string& token : getline_split(s, ',')) {
        if (token == "all") {
            for (int bits = 0; bits < 8; ++bits) combos.push_back(static_cast<uint8_t>(bits));
            continue;
        }
        uint8_t combo = 0;
        if (token != "none") {
            for (const std::string& flag : getline_split(token, '+')) {
                if (flag == "sene") combo |= 1;
                else if (flag == "dent") combo |= 2;
                else if (flag == "et") combo |= 4;
                else
                    fail(SG_INPUT, "unknown improvement '" + flag +
                                       "' (expected sene, dent, et, none or all)");
            }
        }
        combos.push_back(combo);
    }
    if (combos.empty()) fail(SG_INPUT, "empty improvement combination list");
    return combos;
}

int run_sweep(int argc, char** argv) {
    std::string input, format = "tsv", w_list = "32,64", o_rule = "half+1",
                combos = "none,sene+dent+et", report;
    bool json = false, no_timing = false;
    int threads = 1;
    std::vector<int> devices;
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i], v;
        const size_t eq = k.find('=');
        const bool has_eq = k.rfind("--", 0) == 0 && eq != std::string::npos;
        if (has_eq) {
            v = k.substr(eq + 1);
            k = k.substr(0, eq);
        }
        auto val = [&]() -> std::string {
            if (has_eq) return v;
            if (i + 1 >= argc) fail(SG_INPUT, k + " requires a value");
            return argv[++i];
        };
        if (k == "--input") input = val();
        else if (k == "--format") format = val();
        else if (k == "--W-list") w_list = val();
        else if (k == "--O-rule") o_rule = val();
        else if (k == "--combos") combos = val();
        else if (k == "--threads") threads = parse_int(k, val());
        else if (k == "--report") report = val();
        else if (k == "--json") json = true;
        else if (k == "--no-timing") no_timing = true;
        else if (k == "--devices") devices = parse_list(k, val());
        else fail(SG_INPUT, "unknown option '" + k + "'");
    }
    if (input.empty()) fail(SG_INPUT, "--input is required");
    const std::vector<int> Ws = parse_list("--W-list", w_list);
    int o_fixed = -1;
    if (o_rule == "half+1") {
        o_fixed = -1;
    } else if (o_rule.rfind("fixed:", 0) == 0) {
        o_fixed = parse_int("--O-rule", o_rule.substr(6));
    } else {
        fail(SG_INPUT, "unknown O rule '" + o_rule + "'");
    }
    const std::vector<uint8_t> cs = parse_combos(combos);
    (void)threads;  // the GPU path has no CPU worker pool
    int fmt;
    if (format == "tsv") fmt = SG_FORMAT_TSV;
    else if (format == "fasta-pair") fmt = SG_FORMAT_FASTA_PAIR;
    else fail(SG_INPUT, "unknown input format '" + format + "' (expected tsv or fasta-pair)");
    sg_pair_file pf{};
    check(sg_read_pairs(input.c_str(), fmt, &pf));
    sg_sweep_options opt{};
    opt.W_list = Ws.data();
    opt.n_W = static_cast<int32_t>(Ws.size());
    opt.o_fixed = o_fixed;
    opt.combos = cs.data();
    opt.n_combos = static_cast<int32_t>(cs.size());
    sg_scoring_default(&opt.scoring);
    opt.measure_time = !no_timing;
    std::vector<sg_sweep_row> rows(Ws.size() * cs.size());
    const int rc = sg_sweep(&opt, &pf.packed, devices.empty() ? nullptr : devices.data(),
                            static_cast<int>(devices.size()), rows.data());
    sg_pair_file_free(&pf);
    check(rc);
    const int64_t len = sg_sweep_format(rows.data(), static_cast<int64_t>(rows.size()), json, nullptr, 0);
    std::string text(static_cast<size_t>(len) + 1, '\0');
    sg_sweep_format(rows.data(), static_cast<int64_t>(rows.size()), json, &text[0], len + 1);
    text.resize(static_cast<size_t>(len));
    if (json) text += '\n';
    FILE* f = report.empty() || report == "-" ? stdout : std::fopen(report.c_str(), "wb");
    if (!f) fail(SG_INPUT, "cannot write '" + report + "'");
    std::fwrite(text.data(), 1, text.size(), f);
    if (f != stdout) std::fclose(f);
    return 0;
}

int run(int argc, char** argv) {
    if (argc >= 2 && std::strcmp(argv[1], "sweep") == 0) return run_sweep(argc, argv);
    const Args a = parse(argc, argv);
    int format;
    if (a.format == "tsv") format = SG_FORMAT_TSV;  // parse_format, main.cpp:35-39
    else if (a.format == "fasta-pair") format = SG_FORMAT_FASTA_PAIR;
    else fail(SG_INPUT, "unknown input format '" + a.format + "' (expected tsv or fasta-pair)");
    check(sg_validate_config(&a.cfg));
    if (a.threads < 1) fail(SG_CONFIG, "thread count must be at least 1");  // batch.cpp:16
    sg_pair_file pf{};
    check(sg_read_pairs(a.input.c_str(), format, &pf));
    sg_results res{};
    const int rc = sg_align_packed(&a.cfg, &pf.packed, a.devices.empty() ? nullptr : a.devices.data(),
                                   static_cast<int>(a.devices.size()), &res);
    if (rc != SG_OK) {
        std::string msg = sg_last_error();
        // name the pair by its id, as run_batch does (batch.cpp:69-77)
        const std::string key = "pair '";
        if (msg.rfind(key, 0) == 0) {
            const size_t end = msg.find('\'', key.size());
            const long long idx = std::atoll(msg.substr(key.size(), end - key.size()).c_str());
            if (end != std::string::npos && idx >= 0 && idx < pf.n_pairs)
                msg = key + pf.ids[idx] + msg.substr(end);
        }
        sg_pair_file_free(&pf);
        fail(rc, msg);
    }
    const int wrc = sg_write_results(a.output.empty() ? nullptr : a.output.c_str(), &pf, &res, a.json);
    if (wrc == SG_OK && a.cmd == "bench") {  // run_align's report, main.cpp:168-175
        long long windows = 0;
        for (int64_t k = 0; k < res.n_pairs; ++k) windows += res.windows[k];
        const double pps = res.align_seconds > 0 ? res.n_pairs / res.align_seconds : 0.0;
        std::fprintf(stderr,
                     "pairs\t%lld\nthreads\t%d\nseconds\t%g\npairs_per_s\t%g\nwindows\t%lld\n"
                     "stored_bits\t%llu\ntable_writes\t%llu\ntable_reads\t%llu\nrows_computed\t%llu\n"
                     "rows_possible\t%llu\ncells_computed\t%llu\n",
                     static_cast<long long>(res.n_pairs), a.threads, res.align_seconds, pps, windows,
                     (unsigned long long)res.total[SG_CNT_STORED_BITS],
                     (unsigned long long)res.total[SG_CNT_TABLE_WRITES],
                     (unsigned long long)res.total[SG_CNT_TABLE_READS],
                     (unsigned long long)res.total[SG_CNT_ROWS_COMPUTED],
                     (unsigned long long)res.total[SG_CNT_ROWS_POSSIBLE],
                     (unsigned long long)res.total[SG_CNT_CELLS_COMPUTED]);
    }
    std::string werr = wrc == SG_OK ? "" : sg_last_error();
    sg_results_free(&res);
    sg_pair_file_free(&pf);
    if (wrc != SG_OK) fail(wrc, werr);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const CliError& e) {
        if (e.code == SG_INPUT || e.code == SG_CONFIG) {
            std::fprintf(stderr, "error: %s\n", e.msg.c_str());
            return 1;
        }
        std::fprintf(stderr, "internal error: %s\n", e.msg.c_str());
        return 2;
    }
}
