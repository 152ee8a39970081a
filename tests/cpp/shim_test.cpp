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
    return failures ? 1 : 0;
}
