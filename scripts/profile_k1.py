"""Runs K1 on a cfg batch twice (warm-up + profiled launch) for ncu captures."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_09985_b200 as sg

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--pairs", type=int, default=100000)
ap.add_argument("--W", type=int, default=64)
ap.add_argument("--O", type=int, default=24)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--phases", action="store_true", help="per-phase cycle counters")
ap.add_argument("--kernel", default="auto")
a = ap.parse_args()
batch = sg.synth_packed(a.cfg, a.seed, a.pairs)
with sg.options(kernel=a.kernel):
    s = sg.Session(sg.AlignerConfig(W=a.W, O=a.O), batch)
for _ in range(a.runs):
    with sg.options(kernel=a.kernel, diagnostics=2 if a.phases else 0):
        ms, k1 = s.run()
    print(f"cfg{a.cfg} pairs={a.pairs} K1-K3 {ms:.3f} ms  K1 {k1:.3f} ms  {a.pairs / (ms / 1e3):.0f} aln/s  {s.info()}", flush=True)
r = s.fetch()
print("cells_computed", r.total.cells_computed, "ALG_OPS/s (K1)", 4 * ((a.W + 31) // 32) * r.total.cells_computed / (k1 / 1e3) / 1e12, "T")
if a.phases:
    buf = s.phase_cycles()
    for name, o in (("band/K1", 0), ("full", 9)):
        b = buf[o:o + 9]
        tot = b[0] + b[1] + b[2] + b[8]
        if tot == 0: continue
        print(f"{name}: cycles (sum over warps) {tot:.3e}: setup {b[0]/tot:.1%}  DC {b[1]/tot:.1%}  TB {b[2]/tot:.1%}  idle {b[8]/tot:.1%}  chunks {b[3]}  cycles/chunk {(b[0]+b[1]+b[2])/max(b[3],1):.0f}")
        print(f"   lanes in DC per chunk {b[4]/max(b[3],1):.1f}/32  TB trips/chunk {b[5]/max(b[3],1):.1f}  TB lane-steps/entry {b[6]/max(b[7],1):.1f}  TB entries {b[7]}  TB lane-util {b[6]/max(32*b[5],1):.1%}")
    print(f"full warps: STD lane-chunks {buf[18]}  full-frame warp-chunks {buf[19]}  full-frame lane-chunks {buf[20]}")
    print(f"coop: windows {buf[21]}  setup+DC cycles/window {buf[22]/max(buf[21],1):.0f}  TB cycles/window {buf[23]/max(buf[21],1):.0f}  mean D {buf[24]/max(buf[21],1):.1f}")
