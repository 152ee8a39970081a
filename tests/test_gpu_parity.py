"""Parity of the sm_100a path with the reference (through the C ABI).

* Every golden fixture (produced by the unmodified reference, tests/golden/) is
  reproduced exactly: distance, CIGAR (or hash + run count), windows and all
  seven InstrumentationCounters.
* Random and edge-case pairs at many (W, O, switches) match the oracle
  restatement (itself pinned to the same fixtures by test_oracle_pin.py).
* At BASELINE.json's full sizes, size-independent properties hold for every
  pair: the CIGAR replays text -> pattern (validate_replay,
  proj/src/cigar.cpp:70-107), its edit count equals the distance, output is
  deterministic and independent of how pairs are sharded.
"""
import random

import numpy as np
import pytest

import golden_io as G
import oracle_ffi as O

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["auto", "band"])
def frame(request, set_options):
    """Runs a test with the host's choice of K1 kernel and again with the mixed
    band-frame kernel forced: small or short-read batches
    otherwise go to the full-frame K1 (host.cu band_pays)."""
    if request.param == "band":
        set_options(kernel="mixed")
    return request.param


def _cfg(sg, W, Ov, s=1, d=1, e=1):
    return sg.AlignerConfig(W=W, O=Ov, sene=bool(s), dent=bool(d), early_termination=bool(e))


def _compare(res, k, row):
    assert int(res.distance[k]) == row["distance"], row["id"]
    cig = res.cigar_string(k)
    if "cigar" in row:
        assert cig == row["cigar"], row["id"]
    else:
        assert O.fnv1a(cig) == row["hash"], row["id"]
        assert G.run_count(cig) == row["runs"], row["id"]
    assert int(res.windows[k]) == row["windows"], row["id"]
    assert [int(x) for x in res.counters[k]] == row["counters"], row["id"]


@pytest.mark.parametrize("name,W,Ov,s,d,e", G.kat_files())
def test_reference_kats(gpu, frame, name, W, Ov, s, d, e):
    sg = gpu
    pairs = G.kat_pairs()
    rows = G.read_golden(name)
    codes = sg.CodesBatch.from_lists([sg.encode_sequence(pairs[r["id"]][0]) for r in rows],
                                     [sg.encode_sequence(pairs[r["id"]][1]) for r in rows])
    res = sg.align_codes(_cfg(sg, W, Ov, s, d, e), codes)
    for k, row in enumerate(rows):
        _compare(res, k, row)


@pytest.mark.parametrize("name,cfg,W,Ov,s,d,e", G.synth_files())
def test_reference_configs(gpu, frame, name, cfg, W, Ov, s, d, e):
    sg = gpu
    rows = G.read_golden(name)
    first = G.pair_index(rows[0]["id"])
    assert [G.pair_index(r["id"]) for r in rows] == list(range(first, first + len(rows)))
    res = sg.align_packed(_cfg(sg, W, Ov, s, d, e), sg.synth_packed(cfg, first, len(rows)))
    for k, row in enumerate(rows):
        _compare(res, k, row)


def test_reference_doctest_kats(gpu):
    sg = gpu
    # proj/tests/test_aligner.cpp:41-48
    r = sg.align("ACGT", "ACGA", sg.AlignerConfig(W=64, O=33))
    assert (r.distance, sg.cigar_to_string(r.cigar), r.windows) == (1, "3=1X", 1)
    # test_aligner.cpp:30-39: identity of a long pair at three window shapes
    rng = random.Random(41)
    x = "".join(rng.choice("ACGT") for _ in range(10000))
    for W, Ov in ((64, 33), (32, 17), (16, 0)):
        r = sg.align(x, x, sg.AlignerConfig(W=W, O=Ov))
        assert r.distance == 0 and sg.cigar_to_string(r.cigar) == "10000="
    # test_dp.cpp:69-75: non-ACGT never matches
    assert sg.align("ANGT", "ANGT").distance == 1
    assert sg.align("NNNN", "NNNN").distance == 4
    # test_aligner.cpp:67-81: per-window counters accumulate exactly
    y = "".join(rng.choice("ACGT") for _ in range(100))
    r = sg.align(y, y, sg.AlignerConfig(W=64, O=33, sene=True, dent=False))
    assert r.windows == 3 and r.distance == 0
    assert r.counters.rows_computed == 3
    assert r.counters.stored_bits == 2 * 65 * 64 + 39 * 38
    assert r.counters.rows_possible == 3 * 65


def _rand(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(n))


CASES = [(1, 0), (2, 1), (3, 0), (5, 2), (7, 6), (16, 8), (31, 15), (32, 0), (32, 31), (33, 1),
         (40, 20), (63, 62), (64, 0), (64, 24), (64, 33), (64, 63), (65, 33), (96, 40),
         (100, 50), (127, 1), (128, 48), (128, 127),
         # K6 (one warp per pair): windows wider than 128 bits
         (129, 1), (160, 64), (200, 100), (256, 0), (256, 255), (300, 150), (513, 200),
         (1000, 999), (1024, 400)]


@pytest.mark.parametrize("W,Ov", CASES)
def test_random_pairs_match_oracle(gpu, frame, W, Ov):
    """Degenerate and multi-limb windows, N bases, unbalanced and tiny pairs
    (proj/tests/test_aligner.cpp:163-211, acceptance.cpp:244-254)."""
    sg = gpu
    rng = random.Random(W * 1000 + Ov)
    pairs = []
    for k in range(24):
        kind = k % 6
        if kind == 0:
            t, p = _rand(rng, rng.randint(1, 300), "ACGTN"), _rand(rng, rng.randint(1, 300), "ACGTN")
        elif kind == 1:
            t, p = _rand(rng, rng.randint(200, 700)), _rand(rng, rng.randint(1, 40))
        elif kind == 2:
            t, p = _rand(rng, rng.randint(1, 40)), _rand(rng, rng.randint(200, 700))
        elif kind == 3:
            t, p = _rand(rng, rng.randint(1, 3)), _rand(rng, rng.randint(1, 3))
        else:
            t = _rand(rng, rng.randint(100, 1200))
            p = list(t[: len(t) - rng.randint(0, 40)])
            for _ in range(len(p) // 8):
                pos = rng.randrange(len(p))
                c = rng.random()
                if c < 0.4:
                    p[pos] = rng.choice("ACGTN")
                elif c < 0.7:
                    p.insert(pos, rng.choice("ACGT"))
                elif len(p) > 1:
                    del p[pos]
            p = "".join(p)
        pairs.append((t, p))
    combos = [(1, 1, 1), (0, 0, 0), (1, 0, 1), (0, 1, 0)]
    for (s, d, e) in combos:
        codes = sg.CodesBatch.from_lists([sg.encode_sequence(t) for t, _ in pairs],
                                         [sg.encode_sequence(p) for _, p in pairs])
        res = sg.align_codes(_cfg(sg, W, Ov, s, d, e), codes)
        for k, (t, p) in enumerate(pairs):
            a = O.align(O.encode(t), O.encode(p), W=W, O=Ov, sene=s, dent=d, et=e)
            assert int(res.distance[k]) == a.distance, (k, s, d, e)
            assert res.cigar_string(k) == a.cigar, (k, s, d, e)
            assert int(res.windows[k]) == a.windows
            assert [int(x) for x in res.counters[k]] == [a.counters[n] for n in O.COUNTER_NAMES]


WIDE_CROSS = ["kat_W64_O33.tsv", "kat_W16_O0.tsv", "kat_W1_O0.tsv", "kat_W65_O33.tsv",
              "kat_W128_O65.tsv", "kat_W64_O33_s0d0e0.tsv"]


@pytest.mark.parametrize("name", WIDE_CROSS)
def test_wide_kernel_on_narrow_windows(gpu, set_options, name):
    """K6 (csrc/wide_align.cu) forced onto windows K1 normally takes: the same
    reference fixtures must come out (sg_options.kernel = SG_KERNEL_WIDE)."""
    sg = gpu
    W, Ov, s, d, e = next(f[1:] for f in G.kat_files() if f[0] == name)
    set_options(kernel="wide")
    pairs = G.kat_pairs()
    rows = G.read_golden(name)
    codes = sg.CodesBatch.from_lists([sg.encode_sequence(pairs[r["id"]][0]) for r in rows],
                                     [sg.encode_sequence(pairs[r["id"]][1]) for r in rows])
    res = sg.align_codes(_cfg(sg, W, Ov, s, d, e), codes)
    for k, row in enumerate(rows):
        _compare(res, k, row)
    # and on a BASELINE config (cfg2 head: 3000 Illumina-like pairs)
    if name == "kat_W64_O33.tsv":
        rows = G.read_golden("cfg2_head.tsv")
        res = sg.align_packed(_cfg(sg, 64, 24), sg.synth_packed(2, 0, len(rows)))
        for k, row in enumerate(rows):
            _compare(res, k, row)


def test_pairs_within_one_window_are_exact(gpu, frame):
    """test_aligner.cpp:123-133: max(n, m) <= W is aligned exactly (Levenshtein)."""
    sg = gpu
    rng = random.Random(45)
    pairs = [(_rand(rng, rng.randint(1, 64)), _rand(rng, rng.randint(1, 64))) for _ in range(400)]
    codes = sg.CodesBatch.from_lists([sg.encode_sequence(t) for t, _ in pairs],
                                     [sg.encode_sequence(p) for _, p in pairs])
    res = sg.align_codes(sg.AlignerConfig(W=64, O=33), codes)
    for k, (t, p) in enumerate(pairs):
        prev = list(range(len(p) + 1))
        for i in range(1, len(t) + 1):
            cur = [i] + [0] * len(p)
            for j in range(1, len(p) + 1):
                cur[j] = min(prev[j - 1] + (t[i - 1] != p[j - 1]), prev[j] + 1, cur[j - 1] + 1)
            prev = cur
        assert int(res.distance[k]) == prev[-1]


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 5])
def test_full_size_properties(gpu, frame, cfg_id):
    """Every pair of the BASELINE config at full size: the CIGAR replays
    (validate_replay) and its edit count equals the distance; head/tail pairs
    equal the reference's golden vectors."""
    sg = gpu
    codes = sg.synth_codes(cfg_id)
    res = sg.align_codes(sg.AlignerConfig(W=64, O=24), codes)
    assert res.n == codes.n
    assert O.replay_batch(codes, res) == 0
    assert (res.windows > 0).all()
    tl, pl = codes.text_len, codes.pat_len
    assert (res.distance >= np.abs(tl - pl)).all()
    names = {1: ["cfg1_full.tsv"], 2: ["cfg2_head.tsv"], 3: ["cfg3_head.tsv", "cfg3_tail.tsv"],
             5: ["cfg5_head.tsv"]}[cfg_id]
    for name in names:
        for row in G.read_golden(name):
            _compare(res, G.pair_index(row["id"]), row)


def test_cfg4_full_sweep_properties(gpu, frame):
    sg = gpu
    codes = sg.synth_codes(4)
    pk = sg.pack(codes)
    for W, Ov in ((32, 12), (64, 24), (64, 33), (128, 48)):
        res = sg.align_packed(sg.AlignerConfig(W=W, O=Ov), pk)
        assert O.replay_batch(codes, res) == 0
        for row in G.read_golden(f"cfg4_W{W}_O{Ov}.tsv"):
            _compare(res, G.pair_index(row["id"]), row)


def test_sharding_and_determinism(gpu, frame):
    """Output is byte-identical across runs and across shardings of the batch
    (acceptance.cpp:258-281 checks the same across thread counts)."""
    sg = gpu
    pk = sg.synth_packed(5, 0, 3000)
    cfg = sg.AlignerConfig(W=64, O=24)
    a = sg.align_packed(cfg, pk)
    b = sg.align_packed(cfg, pk)
    c = sg.align_packed(cfg, pk, devices=[0, 0, 0])  # three shards, one device
    for r in (b, c):
        assert (r.distance == a.distance).all()
        assert (r.cigar_off == a.cigar_off).all()
        assert bytes(r.runs) == bytes(a.runs)
        assert (r.counters == a.counters).all()


def test_session_matches_one_shot(gpu):
    sg = gpu
    pk = sg.synth_packed(3, 0, 500)
    cfg = sg.AlignerConfig(W=64, O=24)
    one = sg.align_packed(cfg, pk)
    s = sg.Session(cfg, pk)
    for _ in range(2):
        ms, k1 = s.run()
        assert ms > 0 and 0 < k1 <= ms
        r = s.fetch()
        assert (r.distance == one.distance).all() and bytes(r.runs) == bytes(one.runs)
    s.close()


def test_run_batch_api_and_tsv(gpu):
    import io
    sg = gpu
    pairs = [sg.SeqPairRecord("a", "ACGT", "ACGA"), sg.SeqPairRecord("b", "GATTACA", "GATTACA")]
    br = sg.run_batch(pairs, sg.AlignerConfig(), threads=4)
    f = io.StringIO()
    sg.write_batch_tsv(f, pairs, br)
    assert f.getvalue() == "a\t1\t3=1X\nb\t0\t7=\n"
    assert br.gpu_launches >= 1 and br.device_ms > 0
    with pytest.raises(sg.ConfigError):
        sg.run_batch(pairs, sg.AlignerConfig(), threads=0)


@pytest.mark.parametrize("name,k,s,e", G.single_files())
def test_reference_single_window(gpu, name, k, s, e):
    # align_single_window (proj/src/aligner.cpp:87-112), run_batch's found flag
    # (batch.cpp:47-62): exact alignments, "not found" past k, reference counters
    sg = gpu
    pairs = G.single_pairs(name)
    rows = G.read_golden(name)
    cfg = sg.AlignerConfig(W=64, O=33, sene=bool(s), dent=False, early_termination=bool(e),
                           mode="single", k_single=k)
    codes = sg.CodesBatch.from_lists([sg.encode_sequence(pairs[r["id"]][0]) for r in rows],
                                     [sg.encode_sequence(pairs[r["id"]][1]) for r in rows])
    res = sg.align_codes(cfg, codes)
    for j, row in enumerate(rows):
        assert bool(res.found[j]) == (row["distance"] >= 0), row["id"]
        if row["distance"] < 0:
            assert int(res.distance[j]) == -1 and res.cigar_string(j) == "", row["id"]
            assert int(res.windows[j]) == row["windows"], row["id"]
            assert [int(x) for x in res.counters[j]] == row["counters"], row["id"]
        else:
            _compare(res, j, row)


def test_single_window_run_batch_and_tsv(gpu):
    # proj/tests/test_harness.cpp:154-160, test_aligner.cpp:135-161
    sg = gpu
    sw = sg.AlignerConfig(mode="single", dent=False, k_single=2)
    far = [sg.SeqPairRecord("far", "AAAAAAAA", "CCCCCCCC")]
    nf = sg.run_batch(far, sw)
    assert not nf.outcomes[0].found
    import io
    buf = io.StringIO()
    sg.write_batch_tsv(buf, far, nf)
    assert buf.getvalue() == "far\t-1\t*\n"
    cfg = sg.AlignerConfig(mode="single", dent=False, k_single=4)
    r = sg.run_batch([sg.SeqPairRecord("a", "ACGT", "ACGA")], cfg)
    assert r.outcomes[0].found and r.outcomes[0].distance == 1
    assert sg.cigar_to_string(r.outcomes[0].cigar) == "3=1X"
    rng = random.Random(46)
    recs = []
    for k in range(150):
        recs.append(sg.SeqPairRecord(f"p{k}", "".join(rng.choice("ACGT") for _ in range(rng.randint(1, 64))),
                                     "".join(rng.choice("ACGT") for _ in range(rng.randint(1, 64)))))
    res = sg.run_batch(recs, sg.AlignerConfig(mode="single", dent=False, k_single=64))
    for rec, po in zip(recs, res.outcomes):
        assert po.found
        a = O.align(O.encode(rec.text), O.encode(rec.pattern), dent=False, single_window=True,
                    k_single=64)
        assert po.distance == a.distance and sg.cigar_to_string(po.cigar) == a.cigar


@pytest.mark.gpu
def test_mixed_handoffs_terminate(gpu, set_options):
    """K1 mixed: a window the band frame fails on (D > 30) must
    not bounce between the warp roles. For W < 64 a window can be both band- and
    STD-shaped; the W = 32 KATs hit that case (one of them looped for minutes
    when the band frame could take such a window back)."""
    import time
    sg = gpu
    set_options(kernel="mixed")
    pairs = G.kat_pairs()
    rows = G.read_golden("kat_W32_O17.tsv")
    codes = sg.CodesBatch.from_lists([sg.encode_sequence(pairs[r["id"]][0]) for r in rows],
                                     [sg.encode_sequence(pairs[r["id"]][1]) for r in rows])
    sg.align_codes(_cfg(sg, 32, 17, 1, 1, 1), codes)  # warm-up
    for _ in range(3):
        t0 = time.time()
        res = sg.align_codes(_cfg(sg, 32, 17, 1, 1, 1), codes)
        assert time.time() - t0 < 5.0
        for k, row in enumerate(rows):
            _compare(res, k, row)


@pytest.mark.gpu
def test_kernel_choice(gpu):
    """host.cu band_pays: correlated reads longer than a window
    run the mixed kernel (W <= 64, W % 8 == 0); pairs of a single window, batches
    with many unrelated pairs and W = 128 the full frame; W > 128 the wide kernel."""
    sg = gpu
    def kernel(cfg_id, count, W, Ov):
        return sg.Session(sg.AlignerConfig(W=W, O=Ov), sg.synth_packed(cfg_id, 0, count)).info()["kernel"]
    assert kernel(3, 2000, 64, 24) == "mixed"
    assert kernel(4, 500, 64, 33) == "mixed"
    assert kernel(4, 500, 32, 12) == "mixed"
    assert kernel(2, 2000, 64, 24) == "mixed"
    assert kernel(4, 200, 128, 48) == "full"
    assert kernel(5, 2000, 64, 24) == "full"
    assert kernel(4, 200, 256, 96) == "wide"


def _stress_batch(sg, seed, n):
    """Randomized long pairs: correlated reads at 0-25% edits of random mix,
    unrelated pairs, garbage bursts (drifting windows), N bases."""
    rng = np.random.default_rng(seed)
    texts, pats = [], []
    for _ in range(n):
        L = int(np.exp(rng.uniform(np.log(60), np.log(4000))))
        t = list(rng.integers(0, 4, L))
        if rng.random() < 0.08:
            p = list(rng.integers(0, 4, max(1, int(L * rng.uniform(0.5, 1.5)))))
        else:
            rate, mix = rng.uniform(0.0, 0.25), rng.dirichlet([1, 1, 1])
            p = []
            for ch in t[: int(L * rng.uniform(0.85, 1.0))]:
                if rng.random() < rate:
                    kind = rng.choice(3, p=mix)
                    if kind == 0:
                        p.append(int((ch + 1 + rng.integers(3)) % 4))
                    elif kind == 1:
                        p += [int(rng.integers(4)), ch]
                else:
                    p.append(ch)
            if rng.random() < 0.05:
                a = len(p) // 3
                p = p[:a] + list(rng.integers(0, 4, int(rng.integers(30, 200)))) + p[a:]
        if rng.random() < 0.02:
            for _ in range(int(rng.integers(1, 6))):
                t[int(rng.integers(len(t)))] = 4
        texts.append(bytes(t))
        pats.append(bytes(p if p else [0]))
    return texts, pats


@pytest.mark.parametrize("W,Ov,s,d,e", [(64, 24, 1, 1, 1), (64, 33, 0, 0, 0), (48, 16, 1, 0, 1)])
def test_mixed_kernel_matches_full_frame(gpu, W, Ov, s, d, e):
    """K1 mixed (band + STD + cooperative warps, queues, K0 routing) against the
    full-frame K1 on a randomized batch: every distance, CIGAR, window count and
    counter identical; a sample is also checked against the oracle."""
    sg = gpu
    texts, pats = _stress_batch(sg, W * 7 + Ov, 4000)
    codes = sg.CodesBatch.from_lists(texts, pats)
    res = {}
    for fr, kernel in (("band", "mixed"), ("full", "full")):
        with sg.options(kernel=kernel):
            res[fr] = sg.align_codes(_cfg(sg, W, Ov, s, d, e), codes)
    a, b = res["band"], res["full"]
    assert np.array_equal(np.asarray(a.distance), np.asarray(b.distance))
    assert np.array_equal(np.asarray(a.windows), np.asarray(b.windows))
    assert np.array_equal(np.asarray(a.counters), np.asarray(b.counters))
    for k in range(len(texts)):
        assert a.cigar_string(k) == b.cigar_string(k), k
    for k in range(0, len(texts), 80):
        o = O.align(texts[k], pats[k], W=W, O=Ov, sene=s, dent=d, et=e)
        assert int(a.distance[k]) == o.distance and a.cigar_string(k) == o.cigar, k
