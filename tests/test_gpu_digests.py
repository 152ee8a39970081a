"""EVERY pair of every BASELINE config, bit-exact against the reference on the GPU.

tests/golden/digests/ holds, per config and (W, O, switch) setting, an FNV-1a-64
digest of each block of 1,000 pairs' reference results — distance, CIGAR hash, run
count, windows and all 7 InstrumentationCounters (make_digests.py, from the
unmodified run_batch, proj/src/batch.cpp:13-104). This test aligns the whole config
on the GPU (cfg1 10k, cfg2 1M, cfg3 100k, cfg4 20k at 4 (W, O) x 8 switch
combinations, cfg5 500k pairs) and recomputes every block digest from the results
(orc_digest_blocks, pinned on the CPU by test_digests.py). It runs each config with
the host's choice of K1 kernel and again with the mixed kernel forced, so both K1
kernels are checked on every pair (the reference's contract: identical output for
every pair, proj/tests/acceptance.cpp:93-126, :258-281).
"""
import pytest

import golden_io as G
import oracle_ffi as O

pytestmark = pytest.mark.gpu

_BATCH = {}


def _batch(sg, cfg_id):
    if cfg_id not in _BATCH:
        _BATCH.clear()  # one config resident at a time (cfg5 is ~1 GB packed)
        _BATCH[cfg_id] = sg.synth_packed(cfg_id)
    return _BATCH[cfg_id]


@pytest.mark.parametrize("kernel", ["auto", "mixed"])
@pytest.mark.parametrize("name,cfg,W,Ov,s,d,e", G.digest_files())
def test_whole_config_digests(gpu, name, cfg, W, Ov, s, d, e, kernel):
    sg = gpu
    blocks, pairs, total, cells = G.read_digests(name)
    batch = _batch(sg, cfg)
    assert batch.n == pairs
    config = sg.AlignerConfig(W=W, O=Ov, sene=bool(s), dent=bool(d), early_termination=bool(e))
    with sg.options(kernel=kernel):
        res = sg.align_packed(config, batch)
    assert int(res.total.cells_computed) == cells
    got, tot = O.results_digests(res)
    bad = [(b0, cnt) for (b0, cnt, want), have in zip(blocks, got) if want != have]
    assert not bad, f"{name} [{kernel}]: {len(bad)} of {len(blocks)} blocks differ, first {bad[:5]}"
    assert tot == total


def _check_digests(name, res):
    blocks, pairs, total, cells = G.read_digests(name)
    assert int(res.total.cells_computed) == cells
    got, tot = O.results_digests(res)
    bad = [(b0, cnt) for (b0, cnt, want), have in zip(blocks, got) if want != have]
    assert not bad, f"{name}: {len(bad)} of {len(blocks)} blocks differ, first {bad[:5]}"
    assert tot == total


def test_pipelined_launches_cfg3(gpu):
    """One-shot calls of long-read batches run the tail kernels beside K1 mixed, per
    output slice. The same call with SG_DIAG_NO_PIPELINE launches
    them after it: both must reproduce the reference's digests of every pair."""
    sg = gpu
    batch = _batch(sg, 3)
    config = sg.AlignerConfig(W=64, O=24)
    piped = sg.align_packed(config, batch)
    assert piped.gpu_launches > 16, "cfg3 should take the pipelined launches"
    _check_digests("cfg3.tsv", piped)
    with sg.options(diagnostics=8):
        plain = sg.align_packed(config, batch)
    assert plain.gpu_launches <= 8
    _check_digests("cfg3.tsv", plain)
    assert (piped.runs == plain.runs).all() and (piped.cigar_off == plain.cigar_off).all()


def test_pipelined_launches_unrelated_pairs(gpu):
    """cfg5 in input order through the pipelined mixed kernel: pairs of 100..20k bases,
    30 % unrelated — every slice has a tail list and a K0 list (unrelated pairs from
    their start, final windows), and the slices finish out of step."""
    sg = gpu
    batch = _batch(sg, 5)
    with sg.options(kernel="mixed", longest_first=False):
        res = sg.align_packed(sg.AlignerConfig(W=64, O=24), batch)
    assert res.gpu_launches > 16, "cfg5 in input order should take the pipelined launches"
    _check_digests("cfg5.tsv", res)


def test_pipelined_launches_with_n_bases_and_scrambled_pairs(gpu):
    """A long-read batch with non-ACGT bases in some pairs and some patterns replaced by
    unrelated sequence, through the pipelined mixed kernel, the plain launches and the
    full-frame K1: byte-identical output (no reference digests for this batch; the
    full-frame K1 is pinned on the same shapes by the golden fixtures)."""
    import numpy as np
    sg = gpu
    codes = sg.synth_codes(3, 0, 70000)
    text, pat = codes.text.copy(), codes.pattern.copy()
    rng = np.random.default_rng(7)
    for k in rng.choice(codes.n, 3000, replace=False):       # N bases (code 4)
        a, l = int(codes.text_off[k]), int(codes.text_len[k])
        text[a + rng.integers(0, l, 5)] = 4
        b, m = int(codes.pat_off[k]), int(codes.pat_len[k])
        pat[b + rng.integers(0, m, 3)] = 4
    for k in rng.choice(codes.n, 700, replace=False):        # unrelated patterns
        b, m = int(codes.pat_off[k]), int(codes.pat_len[k])
        pat[b:b + m] = rng.integers(0, 4, m, dtype=np.uint8)
    batch = sg.CodesBatch(text, codes.text_off, codes.text_len, pat, codes.pat_off, codes.pat_len)
    config = sg.AlignerConfig(W=64, O=24)
    runs = {}
    for name, opts in (("piped", dict(kernel="mixed")), ("plain", dict(kernel="mixed", diagnostics=8)),
                       ("full", dict(kernel="full"))):
        with sg.options(**opts):
            runs[name] = sg.align_codes(config, batch)
    assert runs["piped"].gpu_launches > 16 and runs["plain"].gpu_launches <= 8
    ref = runs["full"]
    for name in ("piped", "plain"):
        r = runs[name]
        for a, b in ((r.distance, ref.distance), (r.windows, ref.windows), (r.cigar_off, ref.cigar_off),
                     (r.runs, ref.runs), (r.counters, ref.counters)):
            assert np.array_equal(a, b), name
