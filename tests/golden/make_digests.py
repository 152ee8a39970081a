"""Per-block digests of EVERY pair of the five BASELINE configs, from the UNMODIFIED
reference (oracle/_ref/ref_tool digest, i.e. scrooge::run_batch, proj/src/batch.cpp:13-104).

The reference's contract is identical output for every pair, in input order
(proj/tests/acceptance.cpp:93-126, :258-281). Full per-pair fixtures for 1.7 M pairs
would be ~1 GB, so each block of 1,000 consecutive pairs is reduced to one FNV-1a-64
digest of its pairs' records (distance, CIGAR hash, run count, windows, 7 counters;
ref_tool.cpp:digest_line). tests/test_gpu_digests.py recomputes the same digests from
the GPU's results (oracle/genasm_oracle.c:orc_digest_block).

Writes tests/golden/digests/<name>.tsv: `first\\tcount\\tdigest` per block, then
`total\\tpairs\\tdigest\\tcells_computed`. Needs /root/reference (run here, not on the
GPU box). About 40 min on 8 cores; `python make_digests.py cfg3 cfg4_W64_O24_s1d1e1`
regenerates a subset.
"""
from __future__ import annotations

import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
OUT = os.path.join(HERE, "digests")


def jobs():
    """(name, cfg id, W, O, sene, dent, et) for every config × setting BASELINE.json names."""
    out = [("cfg1", 1, 64, 24, 1, 1, 1), ("cfg2", 2, 64, 24, 1, 1, 1),
           ("cfg3", 3, 64, 24, 1, 1, 1), ("cfg5", 5, 64, 24, 1, 1, 1)]
    for (W, O) in [(32, 12), (64, 24), (64, 33), (128, 48)]:
        for bits in range(8):
            s, d, e = bits & 1, (bits >> 1) & 1, (bits >> 2) & 1
            out.append((f"cfg4_W{W}_O{O}_s{s}d{d}e{e}", 4, W, O, s, d, e))
    return out


def main(argv):
    os.makedirs(OUT, exist_ok=True)
    want = set(argv)
    threads = str(os.cpu_count() or 8)
    for name, cfg, W, O, s, d, e in jobs():
        if want and name not in want:
            continue
        path = os.path.join(OUT, name + ".tsv")
        t0 = time.time()
        res = subprocess.run([REF_TOOL, "digest", "--cfg", str(cfg), "--W", str(W), "--O", str(O),
                              "--sene", str(s), "--dent", str(d), "--et", str(e),
                              "--threads", threads], capture_output=True, text=True, check=True)
        with open(path + ".tmp", "w") as f:
            f.write(res.stdout)
        os.replace(path + ".tmp", path)
        print(f"{name}: {res.stdout.splitlines()[-1]}  ({time.time() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
