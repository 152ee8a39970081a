"""The accuracy sweep: run_sweep (proj/src/sweep.cpp:40-107)
with the GPU exact oracle K7 (global_align, proj/src/oracle.cpp:39-89).

CPU tests pin the oracle restatement (orc_global_align, orc_score_cigar,
orc_worst_quantile, and the sweep composed from them) to fixtures made by the
unmodified reference (tests/golden/make_golden.py sweep). GPU tests check
K7 and sg_sweep / `sg_align sweep` against the same fixtures byte for byte.
"""
import os
import random
import subprocess

import pytest

import golden_io as G
import oracle_ffi as O

GOLD = G.HERE


def _pairs(name):
    with open(os.path.join(GOLD, name)) as f:
        return [tuple(line.rstrip("\n").split("\t")) for line in f]


def _global_rows(name):
    out = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            pid, d, cig, score = line.rstrip("\n").split("\t")
            out.append((pid, int(d), cig, int(score)))
    return out


# ---------------------------------------------------------------- CPU: oracle pin

@pytest.mark.parametrize("name", ["sweep_sim", "sweep_mix"])
def test_oracle_global_align_matches_reference(name):
    pairs = {pid: (t, p) for pid, t, p in _pairs(name + ".tsv")}
    for pid, d, cig, score in _global_rows(f"global_{name}.tsv"):
        t, p = pairs[pid]
        assert O.global_align(O.encode(t), O.encode(p)) == (d, cig, score), pid


def test_oracle_quantiles_match_naive():
    # proj/tests/test_harness.cpp:205-222
    rng = random.Random(14)
    import math
    for _ in range(50):
        n = 1 + rng.randrange(500)
        s = [rng.randrange(2001) - 1000 for _ in range(n)]
        for p in (0.5, 0.1, 0.01, 0.001):
            naive = sorted(s)[max(1, math.ceil(p * n)) - 1]
            assert O.worst_quantile(list(s), p) == naive


def _oracle_sweep_csv(pairs, Ws, o_rule, combos):
    """run_sweep composed from the oracle restatements; formatted as sweep_csv."""
    enc = [(O.encode(t), O.encode(p)) for _, t, p in pairs]
    ex = [O.global_align(t, p) for t, p in enc]
    oq = [O.worst_quantile([e[2] for e in ex], q) for q in (0.5, 0.1, 0.01, 0.001)]
    lines = ["W,O,sene,dent,et,q500,q100,q010,q001,frac_optimal,mean_rows_frac,"
             "stored_bits_ratio,pairs_per_s,oracle_q500,oracle_q100,oracle_q010,oracle_q001"]
    for W in Ws:
        Ov = W // 2 + 1 if o_rule is None else o_rule
        for s, d, e in combos:
            rows = rowsp = sb = be = opt = 0
            scores = []
            for (t, p), x in zip(enc, ex):
                a = O.align(t, p, W=W, O=Ov, sene=s, dent=d, et=e)
                runs = [(int(n), op) for n, op in __import__("re").findall(r"(\d+)([=XID])", a.cigar)]
                sc, prev = 0, ""
                for n, op in runs:
                    if op == "=":
                        sc += 2 * n
                    elif op == "X":
                        sc -= 4 * n
                    else:
                        sc -= (2 * n) if op == prev else (4 + 2 * n)
                    prev = op
                scores.append(sc)
                opt += a.distance == x[0]
                rows += a.counters["rows_computed"]
                rowsp += a.counters["rows_possible"]
                sb += a.counters["stored_bits"]
                be += a.counters["baseline_equiv_bits"]
            q = [O.worst_quantile(list(scores), f) for f in (0.5, 0.1, 0.01, 0.001)]
            lines.append(",".join(map(str, [W, Ov, int(s), int(d), int(e), *q])) + "," +
                         ",".join(f"{v:.6f}" for v in (opt / len(enc), rows / rowsp if rowsp else 0.0,
                                                        be / sb if sb else 0.0, 0.0)) + "," +
                         ",".join(map(str, oq)))
    return "\n".join(lines) + "\n"


ALL = [(b & 1, (b >> 1) & 1, (b >> 2) & 1) for b in range(8)]
SWEEPS = [("sweep_sim.tsv", "sweep_sim_default.csv", [32, 64], None, [(0, 0, 0), (1, 1, 1)]),
          ("sweep_mix.tsv", "sweep_mix_all.csv", [32, 64, 128, 200], None, ALL),
          ("sweep_mix.tsv", "sweep_mix_fixed.csv", [48, 96], 20, [(1, 0, 0), (0, 1, 1)])]


@pytest.mark.parametrize("pairs,csv,Ws,o_rule,combos", SWEEPS)
def test_oracle_sweep_matches_reference(pairs, csv, Ws, o_rule, combos):
    with open(os.path.join(GOLD, csv)) as f:
        want = f.read()
    assert _oracle_sweep_csv(_pairs(pairs), Ws, o_rule, combos) == want


def test_score_cigar_kats(sg):
    # proj/tests/test_oracle.cpp:76-89
    f = sg.cigar_from_string
    assert sg.score_cigar(f("10=")) == 20
    assert sg.score_cigar(f("3=1X")) == 2
    assert sg.score_cigar(f("5=2I3=")) == 8
    assert sg.score_cigar(f("2I2=")) == 4 - (4 + 4)
    assert sg.score_cigar(f("1I1D2=")) == 4 - (4 + 2) - (4 + 2)
    with pytest.raises(sg.InputError):
        sg.score_cigar([("Q", 3)])
    with pytest.raises(sg.InputError):
        sg.score_cigar([("=", 0)])


def test_library_quantiles(sg):
    rng = random.Random(15)
    s = [rng.randrange(-500, 500) for _ in range(333)]
    for p in (0.5, 0.1, 0.01, 0.001, 1.0):
        assert sg.worst_quantile(s, p) == O.worst_quantile(list(s), p)
    with pytest.raises(sg.InputError):
        sg.worst_quantile([], 0.5)
    with pytest.raises(sg.InputError):
        sg.worst_quantile([1], 0.0)


def test_sweep_format_csv_and_json(sg):
    rows = [sg.SweepRow(32, 17, False, False, False, 10, -2, -5, -5, 0.75, 1.0, 1.0, 0.0,
                        12, -1, -5, -5),
            sg.SweepRow(64, 33, True, True, True, 10, -2, -5, -5, 0.5, 0.125, 3.5, 12345.5,
                        12, -1, -5, -5)]
    csv = sg.sweep_csv(rows)
    assert csv.splitlines()[1] == "32,17,0,0,0,10,-2,-5,-5,0.750000,1.000000,1.000000,0.000000,12,-1,-5,-5"
    import json
    js = sg.sweep_json(rows)
    assert js.startswith('[\n  {\n    "O": 17,\n    "W": 32,\n    "dent": false,')
    back = json.loads(js)
    assert back[1]["mean_rows_frac"] == 0.125 and back[1]["pairs_per_s"] == 12345.5
    assert '"frac_optimal": 1.0' not in js and '"mean_rows_frac": 1.0' in js
    assert sg.sweep_json([]) == "[]"


# ---------------------------------------------------------------- GPU: K7 and the sweep

@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sweep_sim", "sweep_mix"])
def test_gpu_global_align_matches_reference(gpu, name):
    sg = gpu
    pairs = _pairs(name + ".tsv")
    b = sg.pack(sg.CodesBatch.from_lists([sg.encode_sequence(t) for _, t, _ in pairs],
                                         [sg.encode_sequence(p) for _, _, p in pairs]))
    res = sg.global_align_packed(b)
    want = {r[0]: r for r in _global_rows(f"global_{name}.tsv")}
    for k, (pid, _, _) in enumerate(pairs):
        _, d, cig, score = want[pid]
        assert int(res.distance[k]) == d, pid
        assert res.cigar_string(k) == cig, pid
        assert sg.score_cigar(res.cigar(k)) == score, pid


@pytest.mark.gpu
def test_gpu_global_align_random_against_oracle(gpu, monkeypatch):
    """Edge shapes: empty sides, N bases, patterns over 1024 (several stripes),
    unbalanced pairs; and a tiny batch budget (one pair per launch)."""
    sg = gpu
    rng = random.Random(99)
    texts, pats = [], []
    for k in range(60):
        kind = k % 6
        if kind == 0:
            t, p = rng.randint(0, 3), rng.randint(1, 40)
        elif kind == 1:
            t, p = rng.randint(1, 2500), rng.randint(1, 2500)
        elif kind == 2:
            t, p = rng.randint(1, 60), rng.randint(1000, 3100)
        else:
            t = p = rng.randint(100, 2200)
        a = bytes(rng.randrange(5 if k % 4 == 0 else 4) for _ in range(t))
        b = bytes(rng.randrange(5 if k % 4 == 0 else 4) for _ in range(p))
        if kind >= 3:  # a mutated copy
            b = bytes(x if rng.random() > 0.12 else rng.randrange(4) for x in a if rng.random() > 0.05)
            b = b or b"\x00"
        texts.append(a)
        pats.append(b)
    batch = sg.pack(sg.CodesBatch.from_lists(texts, pats))
    for budget in (None, 1):
        with sg.options(exact_budget=budget):
            res = sg.global_align_packed(batch)
        for k, (t, p) in enumerate(zip(texts, pats)):
            d, cig, score = O.global_align(t, p)
            assert (int(res.distance[k]), res.cigar_string(k)) == (d, cig), (k, len(t), len(p))
            assert sg.score_cigar(res.cigar(k)) == score


@pytest.mark.gpu
@pytest.mark.parametrize("pairs,csv,Ws,o_rule,combos", SWEEPS)
def test_gpu_sweep_matches_reference(gpu, pairs, csv, Ws, o_rule, combos):
    sg = gpu
    recs = [sg.SeqPairRecord(pid, t, p) for pid, t, p in _pairs(pairs)]
    rows = sg.run_sweep(recs, Ws, "half+1" if o_rule is None else f"fixed:{o_rule}",
                        [tuple(c) for c in combos], measure_time=False)
    with open(os.path.join(GOLD, csv)) as f:
        assert sg.sweep_csv(rows) == f.read()


@pytest.mark.gpu
def test_gpu_sweep_cli(gpu, tmp_path):
    """`sg_align sweep` (main.cpp:218-286): byte-identical CSV, JSON, errors."""
    from paper_2208_09985_b200.build import CLI
    inp = os.path.join(GOLD, "sweep_mix.tsv")
    r = subprocess.run([CLI, "sweep", "--input", inp, "--W-list", "32,64,128,200", "--combos", "all",
                        "--no-timing"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    with open(os.path.join(GOLD, "sweep_mix_all.csv")) as f:
        assert r.stdout == f.read()
    out = tmp_path / "rep.json"
    r = subprocess.run([CLI, "sweep", "--input", inp, "--W-list", "48,96", "--O-rule", "fixed:20",
                        "--combos", "sene,dent+et", "--json", "--report", str(out)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    import json
    rows = json.loads(out.read_text())
    with open(os.path.join(GOLD, "sweep_mix_fixed.csv")) as f:
        csv_rows = [line.split(",") for line in f.read().splitlines()[1:]]
    assert [(x["W"], x["O"], x["q500"], x["oracle_q001"]) for x in rows] == \
        [(int(c[0]), int(c[1]), int(c[5]), int(c[16])) for c in csv_rows]
    assert all(x["pairs_per_s"] > 0 for x in rows)
    bad = subprocess.run([CLI, "sweep", "--input", inp, "--combos", "sene+foo"],
                         capture_output=True, text=True)
    assert bad.returncode == 1 and "unknown improvement 'foo'" in bad.stderr
    bad = subprocess.run([CLI, "sweep", "--input", inp, "--O-rule", "third"],
                         capture_output=True, text=True)
    assert bad.returncode == 1 and "unknown O rule 'third'" in bad.stderr
    bad = subprocess.run([CLI, "sweep", "--input", inp, "--W-list", "2000"],
                         capture_output=True, text=True)
    assert bad.returncode == 1 and "window size W out of range" in bad.stderr


@pytest.mark.gpu
def test_gpu_sweep_properties(gpu):
    """test_harness.cpp:224-258: O rule, improvements change footprint never
    scores, single-pair quantiles, byte-identical reports with timing off."""
    sg = gpu
    recs = [sg.SeqPairRecord(pid, t, p) for pid, t, p in _pairs("sweep_sim.tsv")]
    rows = sg.run_sweep(recs, [32, 64], "half+1", ["none", "sene+dent+et"], measure_time=False)
    assert [(r.W, r.O) for r in rows] == [(32, 17), (32, 17), (64, 33), (64, 33)]
    assert rows[2].q500 == rows[3].q500 and rows[2].q001 == rows[3].q001
    assert rows[3].stored_bits_ratio > rows[2].stored_bits_ratio
    assert rows[2].frac_optimal == rows[3].frac_optimal
    single = sg.run_sweep(recs[:1], [32, 64], "half+1", ["none", "sene+dent+et"], measure_time=False)
    for r in single:
        assert r.q500 == r.q001 == r.q100 == r.q010
    again = sg.run_sweep(recs, [32, 64], "half+1", ["none", "sene+dent+et"], measure_time=False)
    assert sg.sweep_csv(rows) == sg.sweep_csv(again)
    with pytest.raises(sg.InputError, match="empty dataset"):
        sg.run_sweep([], [32])
    with pytest.raises(sg.InputError, match="empty W list"):
        sg.run_sweep(recs, [])
    with pytest.raises(sg.ConfigError):
        sg.run_sweep(recs, [64], "fixed:64")
    big = [sg.SeqPairRecord("big", "A" * 100001, "A")]
    with pytest.raises(sg.InputError, match="10\\^5 quadratic-cost guard"):
        sg.run_sweep(big, [64])
