"""Quick GPU-vs-oracle parity check (development aid; the real suite is tests/)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2208_09985_b200 as sg
import oracle_ffi as O

def check(cfg_id, count, W=64, Ov=24, sene=True, dent=True, et=True, first=0):
    b = sg.synth_codes(cfg_id, first, count)
    cfg = sg.AlignerConfig(W=W, O=Ov, sene=sene, dent=dent, early_termination=et)
    t0 = time.time(); r = sg.align_codes(cfg, b); t1 = time.time()
    bad = 0
    for k in range(count):
        t, p = b.pair(k)
        a = O.align(t, p, W=W, O=Ov, sene=sene, dent=dent, et=et)
        g = r.cigar_string(k)
        cnt = [int(x) for x in r.counters[k]]
        ref_cnt = [a.counters[n] for n in O.COUNTER_NAMES]
        if a.distance != r.distance[k] or a.cigar != g or a.windows != r.windows[k] or cnt != ref_cnt:
            bad += 1
            if bad <= 3:
                print(f"  MISMATCH cfg{cfg_id} pair {first+k}: ref d={a.distance} w={a.windows} gpu d={r.distance[k]} w={r.windows[k]}")
                print("   ref", a.cigar[:200]); print("   gpu", g[:200])
                print("   cnt ref", ref_cnt); print("   cnt gpu", cnt)
    print(f"cfg{cfg_id} W={W} O={Ov} s{int(sene)}d{int(dent)}e{int(et)}: {count-bad}/{count} ok  (gpu call {t1-t0:.3f}s, device {r.device_ms:.2f} ms, k1 {r.kernel_ms:.2f} ms)", flush=True)
    return bad

bad = 0
for (t, p, exp) in [("ACGT", "ACGA", "3=1X"), ("GATTACA", "GATTACA", "7="), ("ANGT", "ANGT", None), ("A", "T", "1X")]:
    r = sg.align(t, p, sg.AlignerConfig())
    a = O.align(O.encode(t), O.encode(p), W=64, O=33)
    ok = sg.cigar_to_string(r.cigar) == a.cigar and r.distance == a.distance
    print("KAT", t, p, r.distance, sg.cigar_to_string(r.cigar), "ok" if ok else f"BAD (ref {a.distance} {a.cigar})")
    bad += not ok
bad += check(1, 2000)
bad += check(2, 2000)
bad += check(3, 30)
for (W, Ov) in [(32, 12), (64, 24), (64, 33), (128, 48)]:
    bad += check(4, 10, W, Ov)
    bad += check(4, 5, W, Ov, sene=False, dent=False, et=False)
bad += check(5, 200)
print("TOTAL BAD", bad)
sys.exit(1 if bad else 0)
