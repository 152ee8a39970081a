"""Pins the C oracle (oracle/genasm_oracle.c) to the reference.

Every fixture in tests/golden/ was produced by the unmodified reference
(oracle/_ref/ref_tool over /root/reference/proj/src, see make_golden.py).
The oracle must reproduce each line exactly: distance, CIGAR (or its hash and
run count), window count and all seven InstrumentationCounters.
"""
import pytest

import golden_io as G
import oracle_ffi as O


def _check_row(row, a):
    assert a.distance == row["distance"], row["id"]
    if "cigar" in row:
        assert a.cigar == row["cigar"], row["id"]
    else:
        assert O.fnv1a(a.cigar) == row["hash"], row["id"]
        assert G.run_count(a.cigar) == row["runs"], row["id"]
    assert a.windows == row["windows"], row["id"]
    assert [a.counters[n] for n in G.COUNTERS] == row["counters"], row["id"]


@pytest.mark.parametrize("name,W,Ov,s,d,e", G.kat_files())
def test_oracle_matches_reference_kats(name, W, Ov, s, d, e):
    pairs = G.kat_pairs()
    for row in G.read_golden(name):
        t, p = pairs[row["id"]]
        _check_row(row, O.align(O.encode(t), O.encode(p), W=W, O=Ov, sene=s, dent=d, et=e))


@pytest.mark.parametrize("name,cfg,W,Ov,s,d,e", G.synth_files())
def test_oracle_matches_reference_configs(name, cfg, W, Ov, s, d, e):
    spec = O.baseline_spec(cfg)
    rows = G.read_golden(name)
    if name == "cfg1_full.tsv":
        rows = rows[::7]  # every 7th of 10k keeps the CPU suite fast; the GPU suite checks all
    for row in rows:
        t, p = O.synth_pair(spec, G.pair_index(row["id"]))
        _check_row(row, O.align(t, p, W=W, O=Ov, sene=s, dent=d, et=e))


def test_reference_doctest_kats_on_oracle():
    # proj/tests/test_aligner.cpp:41-48, 30-39, 67-81; test_dp.cpp:69-75
    a = O.align(O.encode("ACGT"), O.encode("ACGA"), W=64, O=33)
    assert (a.distance, a.cigar, a.windows) == (1, "3=1X", 1)
    assert O.align(O.encode("ANGT"), O.encode("ANGT")).distance == 1
    assert O.align(O.encode("NNNN"), O.encode("NNNN")).distance == 4
    import random
    rng = random.Random(48)
    x = bytes(rng.randrange(4) for _ in range(100))
    a = O.align(x, x, W=64, O=33, sene=True, dent=False, et=True)
    assert a.windows == 3 and a.distance == 0
    assert a.counters["rows_computed"] == 3
    assert a.counters["stored_bits"] == 2 * 65 * 64 + 39 * 38
    assert a.counters["rows_possible"] == 3 * 65


def test_oracle_errors():
    with pytest.raises(O.OracleError) as e:
        O.align(O.encode("ACGT"), O.encode("ACGT"), W=32, O=32)
    assert e.value.code == 2  # ConfigError (aligner.cpp:10-12)
    with pytest.raises(O.OracleError) as e:
        O.align(b"", O.encode("ACGT"))
    assert e.value.code == 1  # InputError (aligner.cpp:33)


def test_synth_matches_reference_generator_contract():
    # every BASELINE config generates deterministic pairs of the documented shape
    for cfg, (rmin, rmax) in {1: (100, 100), 2: (250, 250), 3: (10000, 10000),
                              4: (10000, 10000), 5: (100, 20000)}.items():
        spec = O.baseline_spec(cfg)
        assert (spec.read_min, spec.read_max) == (rmin, rmax)
        t1, p1 = O.synth_pair(spec, 7)
        t2, p2 = O.synth_pair(spec, 7)
        assert (t1, p1) == (t2, p2)
        assert set(t1) <= {0, 1, 2, 3} and set(p1) <= {0, 1, 2, 3}
    t, p = O.synth_pair(O.baseline_spec(3), 0)
    assert len(t) == 10500 and 9000 < len(p) < 11000
    t, p = O.synth_pair(O.baseline_spec(1), 0)
    assert len(t) == 110 and p[:3] in (t[:3], p[:3])


@pytest.mark.parametrize("name,k,s,e", G.single_files())
def test_oracle_matches_reference_single_window(name, k, s, e):
    # align_single_window (proj/src/aligner.cpp:87-112): found / not found past k,
    # exact distance and CIGAR, counters taken before the traceback
    pairs = G.single_pairs(name)
    for row in G.read_golden(name):
        t, p = pairs[row["id"]]
        a = O.align(O.encode(t), O.encode(p), W=64, O=33, sene=s, dent=False, et=e,
                    single_window=True, k_single=k)
        _check_row(row, a)
        assert a.found == (row["distance"] >= 0), row["id"]
