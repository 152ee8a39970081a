"""Interleaved A/B timing of K1 under environment-variable variants (development aid).
usage: abtest.py --pairs N --reps K "name:VAR=V,VAR2=W" "name2:..." """
import argparse, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_09985_b200 as sg

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--pairs", type=int, default=100000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("variants", nargs="+")
a = ap.parse_args()
batch = sg.synth_packed(a.cfg, 0, a.pairs)
s = sg.Session(sg.AlignerConfig(W=64, O=24), batch)
vs = []
for v in a.variants:
    name, _, kv = v.partition(":")
    env = dict(x.split("=", 1) for x in kv.split(",") if x)
    vs.append((name, env))
times = {n: [] for n, _ in vs}
s.run()
for r in range(a.reps):
    for name, env in vs:
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        ms, k1 = s.run()
        for k, o in old.items():
            if o is None: os.environ.pop(k, None)
            else: os.environ[k] = o
        times[name].append(k1)
for name, _ in vs:
    t = times[name]
    print(f"{name:20s} K1 median {statistics.median(t):7.2f} ms  min {min(t):7.2f}  max {max(t):7.2f}  ({a.pairs / statistics.median(t) * 1e3 / 1e6:.3f} M aln/s)")
