"""The pair-file readers and result writers against what the
unmodified reference readers (proj/src/io.cpp:66-121) and TSV writer
(proj/src/batch.cpp:106-113) produce on the same files (tests/golden/io/,
made by tests/golden/make_io_golden.py through oracle/_ref/ref_tool)."""
import json
import os
import subprocess

import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
CODE = {c: i for i, c in enumerate("ACGT")}


def _expected(name):
    with open(os.path.join(HERE, name)) as f:
        return f.read().replace("{DIR}/", HERE + "/")


def _codes(s):
    return bytes(CODE.get(ch, 4) for ch in s)


def _check_read(sg, inp, fmt, expected_name):
    exp = _expected(expected_name)
    if exp.startswith("error: "):
        with pytest.raises(sg.InputError) as e:
            sg.read_pairs(inp, fmt)
        assert str(e.value) == exp[len("error: "):].rstrip("\n")
        return
    pf = sg.read_pairs(inp, fmt)
    rows = [l.split("\t") for l in exp.splitlines()]
    assert pf.ids == [r[0] for r in rows]
    for k, (_, t, p) in enumerate(rows):
        assert pf.codes(k) == (_codes(t), _codes(p)), rows[k][0]


@pytest.mark.parametrize("name", ["valid.tsv", "two_fields.tsv", "four_fields.tsv", "empty_id.tsv",
                                  "empty_seq.tsv", "empty_text.tsv", "dup_id.tsv", "empty.tsv",
                                  "missing.tsv"])
def test_tsv_reader_matches_reference(sg, name):
    _check_read(sg, os.path.join(HERE, name), "tsv", name + ".expected")


@pytest.mark.parametrize("a,b,tag", [("text.fa", "pattern.fa", "fa_valid"),
                                     ("text.fa", "short.fa", "fa_count"),
                                     ("unnamed.fa", "pattern.fa", "fa_unnamed"),
                                     ("data_first.fa", "pattern.fa", "fa_data_first"),
                                     ("empty_rec.fa", "pattern.fa", "fa_empty_rec"),
                                     ("dup.fa", "dup.fa", "fa_dup"),
                                     ("text.fa", "missing.fa", "fa_missing")])
def test_fasta_pair_reader_matches_reference(sg, a, b, tag):
    _check_read(sg, os.path.join(HERE, a) + "," + os.path.join(HERE, b), "fasta-pair",
                tag + ".expected")


def test_fasta_pair_needs_two_files(sg):
    _check_read(sg, os.path.join(HERE, "text.fa"), "fasta-pair", "fa_nocomma.expected")


def test_cli_argument_errors():
    from paper_2208_09985_b200.build import CLI
    r = subprocess.run([CLI, "align", "--input", os.path.join(HERE, "valid.tsv"), "--format", "bam"],
                       capture_output=True, text=True)
    assert r.returncode == 1
    assert r.stderr == "error: unknown input format 'bam' (expected tsv or fasta-pair)\n"
    r = subprocess.run([CLI, "align", "--input", os.path.join(HERE, "valid.tsv"), "--mode", "x"],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "unknown mode 'x'" in r.stderr
    r = subprocess.run([CLI, "align", "--input", os.path.join(HERE, "two_fields.tsv")],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "expected exactly 3 tab-separated fields" in r.stderr
    r = subprocess.run([CLI, "align", "--input", os.path.join(HERE, "valid.tsv"), "--threads", "0"],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "thread count must be at least 1" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("inp,args,golden", [
    ("valid.tsv", ["--W", "64", "--O", "33"], "valid_W64_O33.tsv.out"),
    ("valid_short.tsv", ["--mode", "single", "--k", "32"], "valid_short_single_k32.tsv.out")])
def test_cli_tsv_output_matches_reference(gpu, tmp_path, inp, args, golden):
    # run_align's TSV path (main.cpp:152-167) on the reference and on the GPU CLI
    from paper_2208_09985_b200.build import CLI
    out = tmp_path / "out.tsv"
    r = subprocess.run([CLI, "align", "--input", os.path.join(HERE, inp), *args,
                        "--output", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert out.read_text() == _expected(golden)
    # the same pairs as FASTA files give the same lines; JSON carries the same fields
    r = subprocess.run([CLI, "bench", "--input", os.path.join(HERE, inp), *args, "--json"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = json.loads(r.stdout)
    lines = [l.split("\t") for l in _expected(golden).splitlines()]
    assert [(o["id"], o["distance"], o["cigar"]) for o in rows] == \
        [(a, int(b), c) for a, b, c in lines]
    assert list(rows[0].keys()) == ["cigar", "distance", "id", "windows"]
    assert f"pairs\t{len(lines)}\nthreads\t1\n" in r.stderr


@pytest.mark.gpu
def test_read_align_write_roundtrip(gpu, tmp_path):
    sg = gpu
    pf = sg.read_pairs(os.path.join(HERE, "text.fa") + "," + os.path.join(HERE, "pattern.fa"),
                       "fasta-pair")
    res = sg.align_packed(sg.AlignerConfig(), pf.packed)
    out = tmp_path / "o.tsv"
    sg.write_results(str(out), pf, res)
    recs = [sg.SeqPairRecord(i, *[sg.decode_sequence(x) for x in pf.codes(k)])
            for k, i in enumerate(pf.ids)]
    ref = sg.run_batch(recs, sg.AlignerConfig())
    import io
    buf = io.StringIO()
    sg.write_batch_tsv(buf, recs, ref)
    assert out.read_text() == buf.getvalue()
