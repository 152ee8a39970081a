// sg_align: the reference CLI's `align` / `bench` flows (proj/tools/main.cpp:
// 113-177, 287-299) on the GPU path: read pairs (TSV or FASTA pair), align on
// one or more GPUs, write TSV or JSON identical to the reference's output.
//
//   sg_align align --input pairs.tsv [--format tsv|fasta-pair] [--W 64] [--O 33]
//                  [--sene|--no-sene] [--dent|--no-dent] [--et|--no-et]
//                  [--threads N] [--output PATH] [--mode windowed|single] [--k K]
//                  [--json] [--devices 0,1,...]
//   sg_align bench ...same...   (also prints the throughput report on stderr)
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
    if (argc < 2) fail(SG_INPUT, "usage: sg_align align|bench --input FILE [options]");
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

int run(int argc, char** argv) {
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
