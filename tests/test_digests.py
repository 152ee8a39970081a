"""Whole-config digests (tests/golden/digests/, made by make_digests.py from the
UNMODIFIED reference's run_batch, proj/src/batch.cpp:13-104) and the digest
arithmetic itself, pinned on the CPU:

* every BASELINE config and setting has a digest file, with one block per 1,000
  pairs covering every pair, and a total that matches its blocks;
* the digest of cfg1's full per-pair fixture (cigar strings from the reference)
  reproduces the reference's block digests, both in Python and through the C
  digest the GPU test uses (orc_digest_blocks over run bytes);
* the oracle restatement reproduces whole blocks of cfg2 and cfg4.

tests/test_gpu_digests.py then recomputes every digest from the GPU's results.
"""
import numpy as np
import pytest

import golden_io as G
import oracle_ffi as O

EXPECTED = {"cfg1": 10_000, "cfg2": 1_000_000, "cfg3": 100_000, "cfg5": 500_000}
FILES = G.digest_files()


def test_every_config_has_digests():
    names = {f for f, *_ in FILES}
    for cfg in ("cfg1", "cfg2", "cfg3", "cfg5"):
        assert f"{cfg}.tsv" in names
    for W, Ov in ((32, 12), (64, 24), (64, 33), (128, 48)):
        for bits in range(8):
            s, d, e = bits & 1, (bits >> 1) & 1, (bits >> 2) & 1
            assert f"cfg4_W{W}_O{Ov}_s{s}d{d}e{e}.tsv" in names


@pytest.mark.parametrize("name,cfg,W,Ov,s,d,e", FILES)
def test_digest_file_covers_every_pair(name, cfg, W, Ov, s, d, e):
    blocks, pairs, total, cells = G.read_digests(name)
    assert pairs == EXPECTED.get(name[:4], 20_000)
    first = 0
    for b0, cnt, _ in blocks:
        assert b0 == first and 0 < cnt <= 1000
        first += cnt
    assert first == pairs
    assert G.digest_total([h for *_, h in blocks]) == total
    assert cells > 0


def _cfg1_rows():
    return G.read_golden("cfg1_full.tsv")


def _record(r, cigar):
    c = "\t".join(str(x) for x in r["counters"])
    return (f"{r['distance']}\t{O.fnv1a(cigar)}\t{G.run_count(cigar)}\t{r['windows']}\t{c}\n")


def test_cfg1_digest_from_full_fixture_python():
    rows = _cfg1_rows()
    blocks, pairs, total, _ = G.read_digests("cfg1.tsv")
    assert len(rows) == pairs
    got = []
    for b0, cnt, _ in blocks:
        rec = "".join(_record(r, r["cigar"]) for r in rows[b0:b0 + cnt])
        got.append(f"{G.fnv1a_bytes(rec.encode()):016x}")
    assert got == [h for *_, h in blocks]
    assert G.digest_total(got) == total


def test_cfg1_digest_from_run_bytes_c():
    rows = _cfg1_rows()
    blocks, _, total, _ = G.read_digests("cfg1.tsv")
    runs = [O.runs_from_cigar(r["cigar"]) for r in rows]
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in runs])
    got, tot = O.digest_blocks(np.array([r["distance"] for r in rows]),
                               np.array([r["windows"] for r in rows]), None, off,
                               np.frombuffer(b"".join(runs), np.uint8),
                               np.array([r["counters"] for r in rows], np.uint64))
    assert got == [h for *_, h in blocks]
    assert tot == total


def _oracle_block(cfg_id, first, count, W, Ov, s=1, d=1, e=1):
    spec = O.baseline_spec(cfg_id)
    dist, win, cnt, runs = [], [], [], []
    for p in range(first, first + count):
        t, q = O.synth_pair(spec, p)
        a = O.align(t, q, W=W, O=Ov, sene=bool(s), dent=bool(d), et=bool(e))
        dist.append(a.distance)
        win.append(a.windows)
        cnt.append([a.counters[n] for n in O.COUNTER_NAMES])
        runs.append(O.runs_from_cigar(a.cigar))
    off = np.zeros(count + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in runs])
    got, _ = O.digest_blocks(np.array(dist), np.array(win), None, off,
                             np.frombuffer(b"".join(runs), np.uint8), np.array(cnt, np.uint64))
    return got[0]


@pytest.mark.parametrize("name,cfg,block,W,Ov,s,d,e", [
    ("cfg2.tsv", 2, 0, 64, 24, 1, 1, 1),
    ("cfg2.tsv", 2, 999, 64, 24, 1, 1, 1),
])
def test_oracle_reproduces_reference_blocks(name, cfg, block, W, Ov, s, d, e):
    blocks, *_ = G.read_digests(name)
    b0, cnt, want = blocks[block]
    assert _oracle_block(cfg, b0, cnt, W, Ov, s, d, e) == want
