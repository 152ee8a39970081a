// Reference-style checks of the C++ drop-in (include/scrooge_b200.hpp), the
// way proj/tests/test_aligner.cpp and acceptance.cpp use scrooge:: — only the
// namespace differs. Built and run by tests/test_cpp_shim.py on the GPU box.
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>

#include "scrooge_b200.hpp"

using namespace scrooge_b200;

static int failures = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
            ++failures;                                                    \
        }                                                                  \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    Workspace ws;
    AlignerConfig cfg;  // W=64, O=33, all improvements on
    // test_aligner.cpp:41-48
    const AlignmentResult r = align(encode_sequence("ACGT"), encode_sequence("ACGA"), cfg, ws);
    CHECK(r.distance == 1);
    CHECK(cigar_to_string(r.cigar) == "3=1X");
    CHECK(r.windows == 1);
    // test_dp.cpp:69-75 through align
    CHECK(align(encode_sequence("ANGT"), encode_sequence("ANGT"), cfg).distance == 1);
    // identity (test_aligner.cpp:30-39)
    std::string x;
    unsigned s = 41;
    for (int i = 0; i < 10000; ++i) x += "ACGT"[(s = s * 1103515245u + 12345u) >> 30];
    const AlignmentResult id = align(encode_sequence(x), encode_sequence(x), cfg);
    CHECK(id.distance == 0 && cigar_to_string(id.cigar) == "10000=");
    // run_batch + write_batch_tsv (batch.cpp:106-113)
    const std::vector<SeqPairRecord> pairs{{"a", "ACGT", "ACGA"}, {"b", "GATTACA", "GATTACA"}};
    const BatchResult br = run_batch(pairs, cfg, 4);
    std::ostringstream os;
    write_batch_tsv(os, pairs, br);
    CHECK(os.str() == "a\t1\t3=1X\nb\t0\t7=\n");
    CHECK(br.total.rows_computed == br.outcomes[0].counters.rows_computed +
                                        br.outcomes[1].counters.rows_computed);
    // errors (test_aligner.cpp:213-230, test_harness.cpp:160-165)
    AlignerConfig bad;
    bad.W = 32;
    bad.O = 32;
    CHECK(throws<ConfigError>([&] { align(encode_sequence("ACGT"), encode_sequence("ACGT"), bad); }));
    CHECK(throws<InputError>([&] { align(CodeView{}, encode_sequence("ACGT"), cfg); }));
    CHECK(throws<ConfigError>([&] { run_batch(pairs, cfg, 0); }));
    const std::vector<SeqPairRecord> empty_seq{{"e", "", "ACGT"}};
    CHECK(throws<InputError>([&] { run_batch(empty_seq, cfg, 1); }));
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "ok", failures);
    // oracle::global_align / score_cigar (proj/tests/test_oracle.cpp:54-62, 76-89)
    {
        const auto g = oracle::global_align(encode_sequence("ACGT"), encode_sequence("ACGA"));
        CHECK(g.distance == 1 && cigar_to_string(g.cigar) == "3=1X");
        const auto gi = oracle::global_align(encode_sequence("GATTACA"), encode_sequence("GATTACA"));
        CHECK(gi.distance == 0 && cigar_to_string(gi.cigar) == "7=");
        const oracle::ScoringParams sp{2, 4, 4, 2};
        CHECK(oracle::score_cigar({{'=', 5}, {'I', 2}, {'=', 3}}, sp) == 8);
        CHECK(oracle::score_cigar({{'I', 1}, {'D', 1}, {'=', 2}}, sp) == 4 - (4 + 2) - (4 + 2));
        CHECK(throws<InputError>([&] { oracle::score_cigar({{'Q', 3}}, sp); }));
    }
    // run_sweep rows and the O rule (proj/tests/test_harness.cpp:224-258)
    {
        std::vector<SeqPairRecord> sp;
        unsigned t = 7;
        for (int k = 0; k < 8; ++k) {
            std::string a, b;
            for (int i = 0; i < 400; ++i) a += "ACGT"[(t = t * 1103515245u + 12345u) >> 30];
            for (char c : a)
                if (((t = t * 1103515245u + 12345u) >> 27) != 0) b += (t >> 20) % 19 == 0 ? 'A' : c;
            sp.push_back({"s" + std::to_string(k), a, b});
        }
        SweepOptions opt;
        opt.W_list = {32, 64};
        opt.combos = {{false, false, false}, {true, true, true}};
        opt.measure_time = false;
        const SweepReport rep = run_sweep(sp, opt);
        CHECK(rep.rows.size() == 4);
        CHECK(rep.rows[0].W == 32 && rep.rows[0].O == 17 && rep.rows[2].O == 33);
        CHECK(rep.rows[2].q500 == rep.rows[3].q500 && rep.rows[2].q001 == rep.rows[3].q001);
        CHECK(rep.rows[3].stored_bits_ratio > rep.rows[2].stored_bits_ratio);
        CHECK(sweep_csv(rep) == sweep_csv(run_sweep(sp, opt)));
        CHECK(sweep_csv(rep).rfind("W,O,sene,dent,et,q500", 0) == 0);
        CHECK(throws<InputError>([&] { run_sweep({}, opt); }));
        CHECK(worst_quantile({5, 1, 3}, 0.5) == 3);
    }
    return failures ? 1 : 0;
}
