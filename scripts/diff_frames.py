"""Differential stress test (development aid): the mixed band/cooperative K1 against
the full-frame K1 on randomized batches — distances, CIGAR runs, window counts and
counters must be identical. usage: diff_frames.py [seed] [pairs]"""
import os, sys, random
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2208_09985_b200 as sg

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
rng = random.Random(seed)
nrng = np.random.default_rng(seed)

def mutate(s, rate, mix):
    out = []
    for ch in s:
        r = nrng.random()
        if r < rate:
            kind = nrng.choice(3, p=mix)
            if kind == 0: out.append(int((ch + 1 + nrng.integers(3)) % 4))
            elif kind == 1: out.append(int(nrng.integers(4))); out.append(ch)
            # kind 2: deletion
        else:
            out.append(ch)
    return out

texts, pats = [], []
for k in range(n):
    L = int(np.exp(nrng.uniform(np.log(60), np.log(6000))))
    t = list(nrng.integers(0, 4, L))
    kind = nrng.random()
    if kind < 0.08:       # unrelated
        p = list(nrng.integers(0, 4, max(1, int(L * nrng.uniform(0.5, 1.5)))))
    else:
        rate = nrng.uniform(0.0, 0.25)
        mix = nrng.dirichlet([1, 1, 1])
        p = mutate(t[: int(L * nrng.uniform(0.85, 1.0))], rate, mix)
        if nrng.random() < 0.05:  # a burst of garbage in the middle (drifting windows)
            a = len(p) // 3
            p = p[:a] + list(nrng.integers(0, 4, int(nrng.integers(30, 200)))) + p[a:]
    if nrng.random() < 0.02:      # N bases
        for _ in range(int(nrng.integers(1, 6))):
            t[int(nrng.integers(len(t)))] = 4
    texts.append(bytes(t)); pats.append(bytes(p if p else [0]))
batch = sg.CodesBatch.from_lists(texts, pats)
bad = 0
for (W, O) in ((64, 24), (64, 33), (48, 16), (60, 20), (36, 12)):
    for (s_, d_, e_) in ((1, 1, 1), (0, 0, 0), (1, 0, 1)):
        cfg = sg.AlignerConfig(W=W, O=O, sene=bool(s_), dent=bool(d_), early_termination=bool(e_))
        res = {}
        for fr, kern in (("band", "mixed"), ("full", "full")):
            try:
                with sg.options(kernel=kern):
                    res[fr] = sg.align_codes(cfg, batch)
            except Exception as ex:
                res[fr] = ex
        a, b = res["band"], res["full"]
        if isinstance(a, Exception) or isinstance(b, Exception):
            same = type(a) is type(b) and str(a) == str(b)
            print(f"W={W} O={O} s{s_}d{d_}e{e_}: exception band={a!r} full={b!r} {'ok' if same else 'MISMATCH'}")
            bad += not same
            continue
        nd = int(np.sum(np.array(a.distance) != np.array(b.distance)))
        nw = int(np.sum(np.array(a.windows) != np.array(b.windows)))
        nc = int(np.sum(np.array(a.counters) != np.array(b.counters)))
        ncig = sum(a.cigar_string(k) != b.cigar_string(k) for k in range(n)) if nd == 0 else -1
        ok = nd == 0 and nw == 0 and nc == 0 and ncig == 0
        bad += not ok
        print(f"W={W} O={O} s{s_}d{d_}e{e_}: distance {nd} windows {nw} counters {nc} cigars {ncig} -> {'ok' if ok else 'MISMATCH'}", flush=True)
print("TOTAL BAD", bad)
