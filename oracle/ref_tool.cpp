// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Drives the UNMODIFIED reference library (libscrooge_core.a compiled by
// oracle/Makefile from /root/reference/proj/src into oracle/_ref/) through its
// public API: scrooge::align / scrooge::run_batch (proj/include/scrooge/
// aligner.hpp:45, batch.hpp:33-34). Used to (1) produce the golden vectors
// that pin oracle/genasm_oracle.c and the GPU path, and (2) time the
// reference CPU aligner for bench.py --impl reference / cpu_baseline.
//
//   ref_tool align  --input pairs.tsv [cfg flags] [--hash]   per-pair results
//   ref_tool synth  --cfg N --first F --count C [cfg flags] [--hash]
//   ref_tool bench  --cfg N --first F --count C --threads T [cfg flags]
//   ref_tool digest --cfg N [--first F --count C] [--block B] [cfg flags]
//                   per-block FNV-1a digests of every pair's result (see digest_line)
//   ref_tool read --input pairs.tsv | read-fasta --input a.fa,b.fa   parsed pairs
//   ref_tool cli-tsv --input pairs.tsv [cfg flags]   write_batch_tsv output
//   ref_tool simulate --count C --length L --rate R --seed S   simulate_pairs TSV
//   ref_tool global --input pairs.tsv   oracle::global_align + score_cigar per pair
//   ref_tool sweep --input pairs.tsv --W-list 32,64 --O-rule half+1|fixed:N
//                  --combos none,sene+dent+et   run_sweep + sweep_csv (no timing)
// cfg flags: --W w --O o --sene 0|1 --dent 0|1 --et 0|1 --mode windowed|single --k k
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "scrooge/batch.hpp"
#include "scrooge/errors.hpp"
#include "scrooge/io.hpp"
#include "scrooge/oracle.hpp"
#include "scrooge/simulate.hpp"
#include "scrooge/sweep.hpp"
#include <sstream>
#include "synth.h"

namespace {

struct Args {
    std::string cmd, input;
    int cfg = 1;
    long long first = 0, count = -1;
    int threads = 1;
    long long block = 1000;
    bool hash = false;
    int length = 0;
    double rate = 0;
    unsigned long long seed = 0;
    std::string w_list = "32,64", o_rule = "half+1", combos = "none,sene+dent+et";
    scrooge::AlignerConfig config;
};

std::uint64_t fnv1a(const std::string& s) {
    std::uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
    return h;
}

Args parse(int argc, char** argv) {
    Args a;
    if (argc < 2) throw scrooge::InputError("usage: ref_tool align|synth|bench ...");
    a.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw scrooge::InputError("missing value for " + k);
            return argv[++i];
        };
        if (k == "--input") a.input = val();
        else if (k == "--cfg") a.cfg = std::stoi(val());
        else if (k == "--first") a.first = std::stoll(val());
        else if (k == "--count") a.count = std::stoll(val());
        else if (k == "--threads") a.threads = std::stoi(val());
        else if (k == "--hash") a.hash = true;
        else if (k == "--block") a.block = std::stoll(val());
        else if (k == "--length") a.length = std::stoi(val());
        else if (k == "--rate") a.rate = std::stod(val());
        else if (k == "--seed") a.seed = std::stoull(val());
        else if (k == "--W-list") a.w_list = val();
        else if (k == "--O-rule") a.o_rule = val();
        else if (k == "--combos") a.combos = val();
        else if (k == "--W") a.config.W = std::stoi(val());
        else if (k == "--O") a.config.O = std::stoi(val());
        else if (k == "--sene") a.config.sene = std::stoi(val()) != 0;
        else if (k == "--dent") a.config.dent = std::stoi(val()) != 0;
        else if (k == "--et") a.config.early_termination = std::stoi(val()) != 0;
        else if (k == "--k") a.config.k_single = std::stoi(val());
        else if (k == "--mode") {
            const std::string m = val();
            a.config.mode = m == "single" ? scrooge::AlignerConfig::Mode::SingleWindow
                                          : scrooge::AlignerConfig::Mode::Windowed;
        } else throw scrooge::InputError("unknown flag " + k);
    }
    return a;
}

std::vector<scrooge::SeqPairRecord> synth_pairs(const Args& a) {
    sg_synth_spec spec;
    if (!sg_synth_baseline_spec(a.cfg, &spec)) throw scrooge::InputError("bad --cfg");
    const long long count = a.count < 0 ? spec.n_pairs - a.first : a.count;
    std::vector<scrooge::SeqPairRecord> pairs(static_cast<std::size_t>(count));
    const int nt = static_cast<int>(std::min<long long>(16, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            std::vector<std::uint8_t> tb(sg_synth_max_text(&spec)), pb(sg_synth_max_pattern(&spec));
            for (long long q = t; q < count; q += nt) {
                std::int64_t n = 0, m = 0;
                sg_synth_pair(&spec, a.first + q, tb.data(), &n, pb.data(), &m);
                auto& r = pairs[static_cast<std::size_t>(q)];
                r.id = "p" + std::to_string(a.first + q);
                r.text.resize(static_cast<std::size_t>(n));
                r.pattern.resize(static_cast<std::size_t>(m));
                for (std::int64_t i = 0; i < n; ++i) r.text[i] = "ACGT"[tb[i]];
                for (std::int64_t i = 0; i < m; ++i) r.pattern[i] = "ACGT"[pb[i]];
            }
        });
    for (auto& th : pool) th.join();
    return pairs;
}

void print_results(const std::vector<scrooge::SeqPairRecord>& pairs, const scrooge::BatchResult& br,
                   bool hash) {
    for (std::size_t i = 0; i < pairs.size(); ++i) {
        const auto& po = br.outcomes[i];
        const std::string cig = po.found ? scrooge::cigar_to_string(po.cigar) : "*";
        const auto& c = po.counters;
        std::printf("%s\t%lld\t", pairs[i].id.c_str(), static_cast<long long>(po.distance));
        if (hash)
            std::printf("%016llx\t%zu", static_cast<unsigned long long>(fnv1a(cig)), po.cigar.size());
        else
            std::printf("%s", cig.c_str());
        std::printf("\t%d\t%llu\t%llu\t%llu\t%llu\t%llu\t%llu\t%llu\n", po.windows,
                    (unsigned long long)c.stored_bits, (unsigned long long)c.table_writes,
                    (unsigned long long)c.table_reads, (unsigned long long)c.rows_computed,
                    (unsigned long long)c.cells_computed, (unsigned long long)c.rows_possible,
                    (unsigned long long)c.baseline_equiv_bits);
    }
}

// One pair's record in the digest: distance, fnv1a64(cigar_to_string) as 16 hex
// digits, run count, windows, the 7 counters, tab-separated, '\n'-terminated
// ("*" hashes for not-found pairs, as print_results). A block's digest is fnv1a64
// over its pairs' records in input order; the total is fnv1a64 over the block
// digests' 16-hex-digit forms. tests/golden/digest.py and oracle/genasm_oracle.c
// (orc_digest_block) compute the same from the GPU's results.
std::string digest_line(const scrooge::PairOutcome& po) {
    const std::string cig = po.found ? scrooge::cigar_to_string(po.cigar) : "*";
    const auto& c = po.counters;
    char buf[512];
    std::snprintf(buf, sizeof buf, "%lld\t%016llx\t%zu\t%d\t%llu\t%llu\t%llu\t%llu\t%llu\t%llu\t%llu\n",
                  static_cast<long long>(po.distance), static_cast<unsigned long long>(fnv1a(cig)),
                  po.cigar.size(), po.windows, (unsigned long long)c.stored_bits,
                  (unsigned long long)c.table_writes, (unsigned long long)c.table_reads,
                  (unsigned long long)c.rows_computed, (unsigned long long)c.cells_computed,
                  (unsigned long long)c.rows_possible, (unsigned long long)c.baseline_equiv_bits);
    return buf;
}

void run_digest(Args a) {
    sg_synth_spec spec;
    if (!sg_synth_baseline_spec(a.cfg, &spec)) throw scrooge::InputError("bad --cfg");
    const long long first = a.first, count = a.count < 0 ? spec.n_pairs - a.first : a.count;
    const long long chunk = std::max<long long>(a.block, (20000 / a.block) * a.block);
    std::uint64_t total = 1469598103934665603ull;
    std::uint64_t cells = 0;
    for (long long c0 = 0; c0 < count; c0 += chunk) {
        Args sub = a;
        sub.first = first + c0;
        sub.count = std::min(chunk, count - c0);
        const auto pairs = synth_pairs(sub);
        const scrooge::BatchResult br = scrooge::run_batch(pairs, a.config, a.threads);
        for (long long b0 = 0; b0 < sub.count; b0 += a.block) {
            const long long bn = std::min(a.block, sub.count - b0);
            std::string recs;
            for (long long q = b0; q < b0 + bn; ++q) {
                recs += digest_line(br.outcomes[static_cast<std::size_t>(q)]);
                cells += br.outcomes[static_cast<std::size_t>(q)].counters.cells_computed;
            }
            char hex[32];
            std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(fnv1a(recs)));
            for (const char* h = hex; *h; ++h) total = (total ^ static_cast<unsigned char>(*h)) * 1099511628211ull;
            std::printf("%lld\t%lld\t%s\n", sub.first + b0, bn, hex);
        }
        std::fflush(stdout);
    }
    std::printf("total\t%lld\t%016llx\t%llu\n", count, static_cast<unsigned long long>(total),
                static_cast<unsigned long long>(cells));
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Args a = parse(argc, argv);
        if (a.cmd == "align") {
            const auto pairs = scrooge::read_pairs_tsv(a.input);
            print_results(pairs, scrooge::run_batch(pairs, a.config, a.threads), a.hash);
        } else if (a.cmd == "read" || a.cmd == "read-fasta") {
            // the reference readers (io.cpp:66-121): parsed pairs, or the error
            const auto pairs = scrooge::read_pairs(
                a.input, a.cmd == "read" ? scrooge::PairFormat::Tsv : scrooge::PairFormat::FastaPair);
            for (const auto& p : pairs)
                std::printf("%s\t%s\t%s\n", p.id.c_str(), p.text.c_str(), p.pattern.c_str());
        } else if (a.cmd == "cli-tsv") {
            // run_align's TSV output path (main.cpp:152-167): read_pairs, run_batch, write_batch_tsv
            const auto pairs = scrooge::read_pairs(a.input, scrooge::PairFormat::Tsv);
            scrooge::write_batch_tsv(std::cout, pairs, scrooge::run_batch(pairs, a.config, a.threads));
        } else if (a.cmd == "simulate") {
            // simulate_pairs (simulate.hpp:24-31) with the default ErrorMix
            const auto sims = scrooge::simulate_pairs(static_cast<int>(a.count), a.length, a.rate,
                                                      scrooge::ErrorMix{}, a.seed);
            std::vector<scrooge::SeqPairRecord> pairs;
            for (const auto& sp : sims) pairs.push_back(sp.rec);
            scrooge::write_pairs_tsv(std::cout, pairs);
        } else if (a.cmd == "global") {
            const auto pairs = scrooge::read_pairs_tsv(a.input);
            const scrooge::oracle::ScoringParams sp;
            for (const auto& p : pairs) {
                const auto ga = scrooge::oracle::global_align(scrooge::encode_sequence(p.text),
                                                              scrooge::encode_sequence(p.pattern));
                const std::string cig = scrooge::cigar_to_string(ga.cigar);
                std::printf("%s\t%d\t", p.id.c_str(), ga.distance);
                if (a.hash)
                    std::printf("%016llx\t%zu", static_cast<unsigned long long>(fnv1a(cig)),
                                ga.cigar.size());
                else
                    std::printf("%s", cig.c_str());
                std::printf("\t%lld\n", static_cast<long long>(scrooge::oracle::score_cigar(ga.cigar, sp)));
            }
        } else if (a.cmd == "sweep") {
            // the CLI's sweep flow (main.cpp:260-285) with timing off
            scrooge::SweepOptions options;
            std::stringstream ws(a.w_list);
            std::string token;
            while (std::getline(ws, token, ',')) options.W_list.push_back(std::stoi(token));
            if (a.o_rule == "half+1") {
                options.o_rule.kind = scrooge::OverlapRule::Kind::HalfPlusOne;
            } else {
                options.o_rule.kind = scrooge::OverlapRule::Kind::Fixed;
                options.o_rule.fixed = std::stoi(a.o_rule.substr(6));
            }
            std::stringstream cs(a.combos);
            while (std::getline(cs, token, ',')) {
                if (token == "all") {
                    for (int bits = 0; bits < 8; ++bits)
                        options.combos.push_back({(bits & 1) != 0, (bits & 2) != 0, (bits & 4) != 0});
                    continue;
                }
                scrooge::ImprovementCombo combo;
                std::stringstream parts(token);
                std::string flag;
                while (token != "none" && std::getline(parts, flag, '+')) {
                    if (flag == "sene") combo.sene = true;
                    else if (flag == "dent") combo.dent = true;
                    else if (flag == "et") combo.et = true;
                }
                options.combos.push_back(combo);
            }
            options.threads = a.threads;
            options.measure_time = false;
            const auto pairs = scrooge::read_pairs(a.input, scrooge::PairFormat::Tsv);
            std::cout << scrooge::sweep_csv(scrooge::run_sweep(pairs, options));
        } else if (a.cmd == "synth") {
            const auto pairs = synth_pairs(a);
            print_results(pairs, scrooge::run_batch(pairs, a.config, a.threads), a.hash);
        } else if (a.cmd == "digest") {
            run_digest(a);
        } else if (a.cmd == "bench") {
            const auto pairs = synth_pairs(a);
            const scrooge::BatchResult br = scrooge::run_batch(pairs, a.config, a.threads);
            std::uint64_t cells = 0, dsum = 0;
            for (const auto& po : br.outcomes) {
                cells += po.counters.cells_computed;
                dsum += static_cast<std::uint64_t>(po.distance);
            }
            std::printf(
                "{\"pairs\": %zu, \"threads\": %d, \"align_seconds\": %.6f, \"pairs_per_second\": "
                "%.3f, \"cells_computed\": %llu, \"distance_sum\": %llu}\n",
                pairs.size(), a.threads, br.align_seconds, br.pairs_per_second,
                (unsigned long long)cells, (unsigned long long)dsum);
        } else {
            throw scrooge::InputError("unknown command " + a.cmd);
        }
    } catch (const scrooge::InternalError& e) {
        std::fprintf(stderr, "internal error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
