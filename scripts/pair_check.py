"""Per-pair GPU-vs-oracle comparison with window-level detail (development aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2208_09985_b200 as sg
import oracle_ffi as O
cfg_id, count = int(sys.argv[1]), int(sys.argv[2])
b = sg.synth_codes(cfg_id, 0, count)
cfg = sg.AlignerConfig(W=64, O=24)
shown = 0
for k in range(count):
    t, p = b.pair(k)
    a = O.align(t, p, W=64, O=24)
    dopt, nw, mw = O.window_stats()
    one = sg.CodesBatch.from_lists([t], [p]) if hasattr(sg.CodesBatch, "from_lists") else None
    try:
        r = sg.align_codes(cfg, one)
        g, gd = r.cigar_string(0), int(r.distance[0])
        err = None
    except Exception as e:
        g, gd, err = "", -1, str(e)
    if err or g != a.cigar or gd != a.distance:
        shown += 1
        print(f"pair {k}: n={len(t)} m={len(p)} ref d={a.distance} gpu d={gd} err={err}")
        print("  windows d_opt:", list(dopt)[:20], " n_w:", list(nw)[:6], " m_w:", list(mw)[:6])
        if g:
            i = next((x for x in range(min(len(g), len(a.cigar))) if g[x] != a.cigar[x]), 0)
            print("  ref", a.cigar[max(0, i-50):i+40]); print("  gpu", g[max(0, i-50):i+40])
        if shown >= 4: break
print("done")
