"""Regenerates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs oracle/_ref/ref_tool (built by `make -C oracle ref` from
/root/reference/proj/src) — so it only works in a container that has
/root/reference. The fixtures it writes are committed; tests never need the
reference at run time.

Per line: id, distance, cigar (or fnv1a-64 hash + run count for long pairs),
windows, then the 7 InstrumentationCounters (proj/include/scrooge/dp.hpp:46-66).
"""
from __future__ import annotations

import os
import random
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")


def ref(args, out_name):
    res = subprocess.run([REF_TOOL, *args, "--threads", str(os.cpu_count() or 8)],
                         capture_output=True, text=True, check=True)
    with open(os.path.join(HERE, out_name), "w") as f:
        f.write(res.stdout)
    print(out_name, res.stdout.count("\n"), "lines")


def cfg_flags(W, O, sene=1, dent=1, et=1):
    return ["--W", str(W), "--O", str(O), "--sene", str(sene), "--dent", str(dent),
            "--et", str(et)]


def write_pairs(name, pairs):
    with open(os.path.join(HERE, name), "w") as f:
        for pid, t, p in pairs:
            f.write(f"{pid}\t{t}\t{p}\n")


def rand_seq(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(n))


def main():
    if not os.path.exists(REF_TOOL):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)

    # --- reference KATs and edge cases (proj/tests/test_aligner.cpp, test_dp.cpp,
    #     test_traceback.cpp), as TSV pair files
    rng = random.Random(2208)
    x10k = rand_seq(rng, 10000)
    kat = [("acgt_acga", "ACGT", "ACGA"), ("gattaca", "GATTACA", "GATTACA"),
           ("anmt", "ANGT", "ANGT"), ("nnnn", "NNNN", "NNNN"), ("a_t", "A", "T"),
           ("aaaa_cccc", "AAAA", "CCCC"), ("identity10k", x10k, x10k)]
    long_t, short_p = rand_seq(rng, 2000), rand_seq(rng, 40)
    kat += [("unbalanced", long_t, short_p), ("unbalanced_flip", short_p, long_t)]
    for k in range(40):  # pairs inside one window (exact per test_aligner.cpp:123-133)
        kat.append((f"win{k}", rand_seq(rng, rng.randint(1, 64)), rand_seq(rng, rng.randint(1, 64))))
    for k in range(40):  # random pairs with N, lengths 1..300 (test_aligner.cpp:192-211)
        kat.append((f"n{k}", rand_seq(rng, rng.randint(1, 300), "ACGTN"),
                    rand_seq(rng, rng.randint(1, 300), "ACGTN")))
    for k in range(30):  # mutated reads with slack / indels
        base = rand_seq(rng, rng.randint(100, 1500))
        read = list(base[: max(1, len(base) - rng.randint(0, 60))])
        for _ in range(len(read) // 10):
            pos = rng.randrange(len(read))
            r = rng.random()
            if r < 0.4:
                read[pos] = rng.choice("ACGT")
            elif r < 0.7:
                read.insert(pos, rng.choice("ACGT"))
            elif len(read) > 1:
                del read[pos]
        kat.append((f"mut{k}", base, "".join(read)))
    write_pairs("kat_pairs.tsv", kat)
    kat_tsv = os.path.join(HERE, "kat_pairs.tsv")
    for (W, O) in [(64, 33), (32, 17), (16, 0), (4, 3), (1, 0), (2, 1), (3, 2), (5, 3), (31, 30),
                   (33, 17), (63, 0), (65, 33), (96, 40), (127, 64), (128, 65), (64, 63)]:
        ref(["align", "--input", kat_tsv, *cfg_flags(W, O)], f"kat_W{W}_O{O}.tsv")
    ref(["align", "--input", kat_tsv, *cfg_flags(64, 33, 0, 0, 0)], "kat_W64_O33_s0d0e0.tsv")
    ref(["align", "--input", kat_tsv, *cfg_flags(64, 33, 1, 0, 1)], "kat_W64_O33_s1d0e1.tsv")

    # --- BASELINE configs (seeded synthetic pairs, paper_2208_09985_b200/csrc/synth.c)
    ref(["synth", "--cfg", "1", "--count", "10000", *cfg_flags(64, 24)], "cfg1_full.tsv")
    ref(["synth", "--cfg", "2", "--count", "3000", *cfg_flags(64, 24)], "cfg2_head.tsv")
    ref(["synth", "--cfg", "3", "--count", "300", "--hash", *cfg_flags(64, 24)], "cfg3_head.tsv")
    ref(["synth", "--cfg", "3", "--first", "99900", "--count", "100", "--hash",
         *cfg_flags(64, 24)], "cfg3_tail.tsv")
    for (W, O) in [(32, 12), (64, 24), (64, 33), (128, 48)]:
        ref(["synth", "--cfg", "4", "--count", "40", "--hash", *cfg_flags(W, O)],
            f"cfg4_W{W}_O{O}.tsv")
        for bits in range(8):
            s, d, e = bits & 1, (bits >> 1) & 1, (bits >> 2) & 1
            ref(["synth", "--cfg", "4", "--first", "1000", "--count", "6", "--hash",
                 *cfg_flags(W, O, s, d, e)], f"cfg4_W{W}_O{O}_s{s}d{d}e{e}.tsv")
    ref(["synth", "--cfg", "5", "--count", "500", "--hash", *cfg_flags(64, 24)], "cfg5_head.tsv")

    # --- single-window mode (align_single_window, proj/src/aligner.cpp:87-112;
    #     proj/tests/test_aligner.cpp:135-161, test_harness.cpp:154-160)
    rng = random.Random(8712)
    single = [("acgt_acga", "ACGT", "ACGA"), ("gattaca", "GATTACA", "GATTACA"),
              ("aaaa_cccc", "AAAA", "CCCC"), ("far", "AAAAAAAA", "CCCCCCCC"),
              ("anmt", "ANGT", "ANGT"), ("a_t", "A", "T")]
    for k in range(60):  # random pairs, lengths 1..128, with N
        single.append((f"r{k}", rand_seq(rng, rng.randint(1, 128), "ACGTN" if k % 5 == 0 else "ACGT"),
                       rand_seq(rng, rng.randint(1, 128))))
    for k in range(40):  # related pairs (a read and its mutated copy), lengths up to 128
        base = rand_seq(rng, rng.randint(1, 120))
        read = list(base)
        for _ in range(max(1, len(read) // 8)):
            pos = rng.randrange(len(read))
            r = rng.random()
            if r < 0.4:
                read[pos] = rng.choice("ACGT")
            elif r < 0.7:
                read.insert(pos, rng.choice("ACGT"))
            elif len(read) > 1:
                del read[pos]
        single.append((f"m{k}", base, "".join(read)))
    write_pairs("single_pairs.tsv", single)
    single_tsv = os.path.join(HERE, "single_pairs.tsv")
    for k in (0, 2, 3, 16, 64, 128, 1024):
        for s, e in ((1, 1), (0, 1), (1, 0), (0, 0)):
            ref(["align", "--input", single_tsv, "--mode", "single", "--k", str(k),
                 "--W", "64", "--O", "33", "--sene", str(s), "--dent", "0", "--et", str(e)],
                f"single_k{k}_s{s}e{e}.tsv")

    wide()


def wide():
    """Windows wider than 128 bits (K6): W up to 1024 (AlignerConfig::validate,
    proj/src/aligner.cpp:8-18) and single windows of up to 1024 characters."""
    if not os.path.exists(REF_TOOL):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    kat_tsv = os.path.join(HERE, "kat_pairs.tsv")
    for (W, O) in [(129, 64), (200, 199), (256, 100), (512, 200), (1024, 400), (1024, 0)]:
        ref(["align", "--input", kat_tsv, *cfg_flags(W, O)], f"kat_W{W}_O{O}.tsv")
    ref(["align", "--input", kat_tsv, *cfg_flags(256, 100, 0, 0, 0)], "kat_W256_O100_s0d0e0.tsv")
    ref(["synth", "--cfg", "4", "--count", "12", "--hash", *cfg_flags(256, 96)], "cfg4_W256_O96.tsv")
    for bits in (0, 3, 5, 7):
        s, d, e = bits & 1, (bits >> 1) & 1, (bits >> 2) & 1
        ref(["synth", "--cfg", "4", "--first", "1000", "--count", "3", "--hash",
             *cfg_flags(256, 96, s, d, e)], f"cfg4_W256_O96_s{s}d{d}e{e}.tsv")
    ref(["synth", "--cfg", "4", "--count", "4", "--hash", *cfg_flags(1024, 400)],
        "cfg4_W1024_O400.tsv")

    rng = random.Random(8713)
    single = [("acgt_acga", "ACGT", "ACGA"), ("far", "AAAAAAAA", "CCCCCCCC")]
    for k in range(24):  # random pairs, lengths up to 1024, some with N
        single.append((f"r{k}", rand_seq(rng, rng.randint(100, 1024), "ACGTN" if k % 6 == 0 else "ACGT"),
                       rand_seq(rng, rng.randint(100, 1024))))
    for k in range(36):  # a read and its mutated copy
        base = rand_seq(rng, rng.randint(129, 1000))
        read = list(base)
        for _ in range(max(1, len(read) // rng.choice((6, 12, 40)))):
            pos = rng.randrange(len(read))
            r = rng.random()
            if r < 0.4:
                read[pos] = rng.choice("ACGT")
            elif r < 0.7:
                read.insert(pos, rng.choice("ACGT"))
            elif len(read) > 1:
                del read[pos]
        single.append((f"m{k}", base, "".join(read)[:1024]))
    single.append(("max", rand_seq(rng, 1024), rand_seq(rng, 1024)))
    write_pairs("single_wide_pairs.tsv", single)
    single_tsv = os.path.join(HERE, "single_wide_pairs.tsv")
    for k in (16, 300, 1024):
        for s, e in ((1, 1), (0, 0)):
            ref(["align", "--input", single_tsv, "--mode", "single", "--k", str(k),
                 "--W", "64", "--O", "33", "--sene", str(s), "--dent", "0", "--et", str(e)],
                f"single_wide_k{k}_s{s}e{e}.tsv")

    sweep()


def sweep():
    """The accuracy sweep (run_sweep, proj/src/sweep.cpp:40-107) and its exact
    oracle (global_align / score_cigar, proj/src/oracle.cpp:39-115)."""
    if not os.path.exists(REF_TOOL):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)

    def sim(count, length, rate, seed):
        res = subprocess.run([REF_TOOL, "simulate", "--count", str(count), "--length", str(length),
                              "--rate", str(rate), "--seed", str(seed)],
                             capture_output=True, text=True, check=True)
        return [tuple(line.split("\t")) for line in res.stdout.splitlines()]

    # proj/tests/test_harness.cpp:224-258's dataset
    write_pairs("sweep_sim.tsv", sim(8, 400, 0.05, 15))
    # a harder mix: long reads (multi-stripe patterns), high error, N bases, tiny pairs
    rng = random.Random(4242)
    mix = sim(24, 1500, 0.1, 77) + [(f"l{k}", t, p) for k, (_, t, p) in enumerate(sim(4, 3000, 0.15, 78))]
    for k in range(8):
        mix.append((f"n{k}", rand_seq(rng, rng.randint(1, 200), "ACGTN"),
                    rand_seq(rng, rng.randint(1, 200), "ACGTN")))
    mix += [("tiny", "A", "T"), ("one", "ACGT", "ACGA"), ("unb", rand_seq(rng, 900), rand_seq(rng, 30))]
    write_pairs("sweep_mix.tsv", mix)
    for name in ("sweep_sim", "sweep_mix"):
        tsv = os.path.join(HERE, name + ".tsv")
        ref(["global", "--input", tsv], f"global_{name}.tsv")
    sim_tsv, mix_tsv = os.path.join(HERE, "sweep_sim.tsv"), os.path.join(HERE, "sweep_mix.tsv")
    ref(["sweep", "--input", sim_tsv], "sweep_sim_default.csv")
    ref(["sweep", "--input", mix_tsv, "--W-list", "32,64,128,200", "--combos", "all"],
        "sweep_mix_all.csv")
    ref(["sweep", "--input", mix_tsv, "--W-list", "48,96", "--O-rule", "fixed:20",
         "--combos", "sene,dent+et"], "sweep_mix_fixed.csv")


if __name__ == "__main__":
    if sys.argv[1:] == ["wide"]:
        sys.exit(wide())
    if sys.argv[1:] == ["sweep"]:
        sys.exit(sweep())
    sys.exit(main())
