"""Small GPU-vs-oracle parity check of one config (development aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2208_09985_b200 as sg
import oracle_ffi as O
cfg_id, count = int(sys.argv[1]), int(sys.argv[2])
W = int(sys.argv[3]) if len(sys.argv) > 3 else 64
Ov = int(sys.argv[4]) if len(sys.argv) > 4 else 24
b = sg.synth_codes(cfg_id, 0, count)
cfg = sg.AlignerConfig(W=W, O=Ov)
try:
    r = sg.align_codes(cfg, b)
except Exception as e:
    print("ERROR", e); sys.exit(1)
bad = 0
for k in range(count):
    t, p = b.pair(k)
    a = O.align(t, p, W=W, O=Ov)
    if a.distance != r.distance[k] or a.cigar != r.cigar_string(k) or a.windows != r.windows[k]:
        bad += 1
        if bad <= 2:
            print(f" pair {k}: ref d={a.distance} w={a.windows} gpu d={r.distance[k]} w={r.windows[k]}")
            ra, ga = a.cigar, r.cigar_string(k)
            i = next((x for x in range(min(len(ra), len(ga))) if ra[x] != ga[x]), min(len(ra), len(ga)))
            print("   ref", ra[max(0,i-60):i+60]); print("   gpu", ga[max(0,i-60):i+60])
print(f"cfg{cfg_id} {os.environ.get('SG_BAND_ROWS','-')} {os.environ.get('SG_J_DIV','-')}: {count-bad}/{count} ok")
