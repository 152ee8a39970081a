"""Regenerates tests/golden/io/: pair-file inputs (valid and malformed) and what
the UNMODIFIED reference readers and TSV writer make of them (oracle/_ref/ref_tool
read / read-fasta / cli-tsv over proj/src/io.cpp and batch.cpp). Needs
/root/reference; the outputs are committed."""
from __future__ import annotations

import os
import random
import subprocess
import sys

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")


def w(name, data: bytes):
    with open(os.path.join(HERE, name), "wb") as f:
        f.write(data)


def ref(cmd, inp, out_name, extra=()):
    r = subprocess.run([REF_TOOL, cmd, "--input", inp, *extra], capture_output=True, text=True)
    with open(os.path.join(HERE, out_name), "w") as f:
        if r.returncode == 0:
            f.write(r.stdout)
        else:
            f.write(r.stderr.replace(HERE + "/", "{DIR}/"))  # "error: <message>"
    print(out_name, r.returncode)


def main():
    os.makedirs(HERE, exist_ok=True)
    rng = random.Random(6611)
    seq = lambda n, a="ACGT": "".join(rng.choice(a) for _ in range(n))
    lines = [f"p{k}\t{seq(rng.randint(1, 150))}\t{seq(rng.randint(1, 150))}" for k in range(40)]
    lines += ["low\tacgtnacgt\tACGTTacg", "iupac\tACGRYKMSWN\tACGT", "x y\tAC GT\tACGT"]
    valid = "\n".join(lines[:10]) + "\n\n" + "\r\n".join(lines[10:25]) + "\r\n\r\n" + "\n".join(lines[25:])
    w("valid.tsv", valid.encode())  # no final newline, CRLF block, empty lines
    short = [l for l in lines if max(len(x) for x in l.split("\t")[1:]) <= 128]
    w("valid_short.tsv", ("\n".join(short) + "\n").encode())  # single-window GPU limit 128
    w("two_fields.tsv", b"a\tACGT\tACGT\nb\tACGT\n")
    w("four_fields.tsv", b"a\tACGT\tACGT\tX\n")
    w("empty_id.tsv", b"a\tACGT\tACGT\n\tACGT\tACGT\n")
    w("empty_seq.tsv", b"a\tACGT\t\n")
    w("empty_text.tsv", b"a\t\tACGT\n")
    w("dup_id.tsv", b"a\tACGT\tACGT\nb\tA\tA\na\tC\tC\n")
    w("empty.tsv", b"")
    recs_t = [(f"r{k}", seq(rng.randint(1, 200))) for k in range(20)]
    recs_p = [(f"q{k}", seq(rng.randint(1, 200))) for k in range(20)]
    def fasta(recs, width=60, desc=True):
        out = []
        for i, (name, s) in enumerate(recs):
            out.append(f">{name}" + (f" sample description {i}" if desc and i % 2 else ""))
            for j in range(0, len(s), width):
                out.append(s[j:j + width].lower() if i % 3 == 0 else s[j:j + width])
        return "\n".join(out) + "\n"
    w("text.fa", fasta(recs_t).encode())
    w("pattern.fa", fasta(recs_p, 50, False).replace("\n", "\r\n").encode())
    w("short.fa", fasta(recs_p[:5]).encode())
    w("unnamed.fa", b">r0\nACGT\n> x\nACGT\n")
    w("data_first.fa", b"ACGT\n>r0\nACGT\n")
    w("empty_rec.fa", b">r0\nACGT\n>r1\n>r2\nAC\n")
    w("dup.fa", b">r0\nACGT\n>r0\nACGT\n")
    d = lambda n: os.path.join(HERE, n)
    for name in ["valid.tsv", "two_fields.tsv", "four_fields.tsv", "empty_id.tsv", "empty_seq.tsv",
                 "empty_text.tsv", "dup_id.tsv", "empty.tsv", "missing.tsv"]:
        ref("read", d(name), name + ".expected")
    for a, b, tag in [("text.fa", "pattern.fa", "fa_valid"), ("text.fa", "short.fa", "fa_count"),
                      ("unnamed.fa", "pattern.fa", "fa_unnamed"),
                      ("data_first.fa", "pattern.fa", "fa_data_first"),
                      ("empty_rec.fa", "pattern.fa", "fa_empty_rec"),
                      ("dup.fa", "dup.fa", "fa_dup"), ("text.fa", "missing.fa", "fa_missing")]:
        ref("read-fasta", d(a) + "," + d(b), tag + ".expected")
    ref("read-fasta", d("text.fa"), "fa_nocomma.expected")
    ref("cli-tsv", d("valid.tsv"), "valid_W64_O33.tsv.out", ("--W", "64", "--O", "33"))
    ref("cli-tsv", d("valid_short.tsv"), "valid_short_single_k32.tsv.out",
        ("--mode", "single", "--k", "32", "--dent", "0"))


if __name__ == "__main__":
    sys.exit(main())
