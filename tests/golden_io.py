"""Readers for the reference-generated fixtures in tests/golden/ (see make_golden.py)."""
from __future__ import annotations

import glob
import os
import re

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
COUNTERS = ("stored_bits", "table_writes", "table_reads", "rows_computed", "cells_computed",
            "rows_possible", "baseline_equiv_bits")


def read_golden(name):
    rows = []
    with open(os.path.join(HERE, name)) as f:
        for line in f:
            parts = line.rstrip("\n").split("\t")
            hashed = len(parts) == 12
            r = {"id": parts[0], "distance": int(parts[1])}
            if hashed:
                r["hash"], r["runs"] = parts[2], int(parts[3])
                rest = parts[4:]
            else:
                r["cigar"] = parts[2]
                rest = parts[3:]
            r["windows"] = int(rest[0])
            r["counters"] = [int(x) for x in rest[1:8]]
            rows.append(r)
    return rows


def kat_pairs():
    out = {}
    with open(os.path.join(HERE, "kat_pairs.tsv")) as f:
        for line in f:
            pid, t, p = line.rstrip("\n").split("\t")
            out[pid] = (t, p)
    return out


_KAT = re.compile(r"kat_W(\d+)_O(\d+)(?:_s(\d)d(\d)e(\d))?\.tsv$")
_CFG4 = re.compile(r"cfg4_W(\d+)_O(\d+)(?:_s(\d)d(\d)e(\d))?\.tsv$")


def kat_files():
    """(file, W, O, sene, dent, et) of every KAT result file."""
    out = []
    for path in sorted(glob.glob(os.path.join(HERE, "kat_W*.tsv"))):
        m = _KAT.search(path)
        s, d, e = (int(m.group(3)), int(m.group(4)), int(m.group(5))) if m.group(3) else (1, 1, 1)
        out.append((os.path.basename(path), int(m.group(1)), int(m.group(2)), s, d, e))
    return out


def synth_files():
    """(file, cfg_id, W, O, sene, dent, et) of every synthetic-config file."""
    out = [("cfg1_full.tsv", 1, 64, 24, 1, 1, 1), ("cfg2_head.tsv", 2, 64, 24, 1, 1, 1),
           ("cfg3_head.tsv", 3, 64, 24, 1, 1, 1), ("cfg3_tail.tsv", 3, 64, 24, 1, 1, 1),
           ("cfg5_head.tsv", 5, 64, 24, 1, 1, 1)]
    for path in sorted(glob.glob(os.path.join(HERE, "cfg4_W*.tsv"))):
        m = _CFG4.search(path)
        s, d, e = (int(m.group(3)), int(m.group(4)), int(m.group(5))) if m.group(3) else (1, 1, 1)
        out.append((os.path.basename(path), 4, int(m.group(1)), int(m.group(2)), s, d, e))
    return out


def pair_index(pid: str) -> int:
    return int(pid[1:])


def run_count(cigar: str) -> int:
    return len(re.findall(r"\d+[=XID]", cigar))


_SINGLE = re.compile(r"single_(wide_)?k(\d+)_s(\d)e(\d)\.tsv$")


def single_pairs(name="single_k0_s1e1.tsv"):
    """Pairs of a single-window result file: single_pairs.tsv (lengths <= 128)
    or single_wide_pairs.tsv (lengths up to 1024)."""
    src = "single_wide_pairs.tsv" if name.startswith("single_wide_") else "single_pairs.tsv"
    out = {}
    with open(os.path.join(HERE, src)) as f:
        for line in f:
            pid, t, p = line.rstrip("\n").split("\t")
            out[pid] = (t, p)
    return out


def single_files():
    """(file, k_single, sene, et) of every single-window result file (dent off)."""
    out = []
    for path in sorted(glob.glob(os.path.join(HERE, "single_*k*_s*e*.tsv"))):
        m = _SINGLE.search(path)
        out.append((os.path.basename(path), int(m.group(2)), int(m.group(3)), int(m.group(4))))
    return out


_DIGEST = re.compile(r"(cfg\d)(?:_W(\d+)_O(\d+)_s(\d)d(\d)e(\d))?\.tsv$")


def digest_files():
    """(file, cfg_id, W, O, sene, dent, et) of every whole-config digest file
    (tests/golden/make_digests.py)."""
    out = []
    for path in sorted(glob.glob(os.path.join(HERE, "digests", "cfg*.tsv"))):
        m = _DIGEST.search(path)
        cfg = int(m.group(1)[3:])
        if m.group(2):
            W, O, s, d, e = (int(m.group(k)) for k in range(2, 7))
        else:
            W, O, s, d, e = 64, 24, 1, 1, 1
        out.append((os.path.basename(path), cfg, W, O, s, d, e))
    return out


def read_digests(name):
    """-> (blocks [(first, count, hex)], total_pairs, total_hex, total_cells)."""
    blocks, total = [], None
    with open(os.path.join(HERE, "digests", name)) as f:
        for line in f:
            parts = line.rstrip("\n").split("\t")
            if parts[0] == "total":
                total = (int(parts[1]), parts[2], int(parts[3]))
            else:
                blocks.append((int(parts[0]), int(parts[1]), parts[2]))
    assert total is not None, name
    return blocks, total[0], total[1], total[2]


def fnv1a_bytes(b: bytes, h: int = 1469598103934665603) -> int:
    for ch in b:
        h = ((h ^ ch) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def digest_total(block_hex):
    """The digest file's total: fnv1a64 over the blocks' 16-hex-digit forms."""
    return f"{fnv1a_bytes(''.join(block_hex).encode()):016x}"
