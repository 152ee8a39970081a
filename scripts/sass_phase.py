"""Attributes an ncu source-page SASS CSV (--page source --csv --print-source sass)
to K1 phases via nvdisasm line info. Development aid.
usage: sass_phase.py <nvdisasm -g -c output> <ncu csv> <kernel L>"""
import csv, re, sys
from collections import defaultdict

dis, csvp, L = sys.argv[1], sys.argv[2], sys.argv[3]
sec = f"k1_window_alignILi{L}E"
addr_line, cur, inside = {}, None, False
for ln in open(dis):
    if ".text." in ln and "//---" in ln:
        inside = sec in ln
        continue
    if not inside:
        continue
    m = re.search(r'line (\d+)', ln)
    if "//## File" in ln and m:
        cur = int(m.group(1)); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur is not None:
        addr_line[int(m.group(1), 16)] = cur

def phase(l):
    if l is None: return "?"
    if 187 <= l <= 275 or 316 <= l <= 453 or 765 <= l <= 771 or l in (155, 156, 157, 158, 161, 162, 163, 164): return "DC"
    if 521 <= l <= 545 or 711 <= l <= 732 or 773 <= l <= 872: return "TB"
    if 546 <= l <= 710 or 736 <= l <= 762 or l < 155: return "setup"
    return f"other"

rows = list(csv.reader(open(csvp)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
H = rows[hdr]
ix = {k: H.index(k) for k in H}
data = [r for r in rows[hdr + 1:] if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
agg = defaultdict(lambda: defaultdict(float))
stall_cols = [k for k in H if k.startswith("stall_") and "Not Issued" not in k]
for r in data:
    off = int(r[0], 16) - base
    ph = phase(addr_line.get(off))
    a = agg[ph]
    a["samples"] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    a["inst"] += float(r[ix["Instructions Executed"]] or 0)
    a["thr"] += float(r[ix["Thread Instructions Executed"]] or 0)
    for k in stall_cols:
        a[k] += float(r[ix[k]] or 0)
tot_s = sum(a["samples"] for a in agg.values()); tot_i = sum(a["inst"] for a in agg.values())
for ph, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"]):
    top = sorted(((a[k], k[6:]) for k in stall_cols), reverse=True)[:6]
    print(f"{ph:6s} samples {a['samples']/tot_s:6.1%}  inst {a['inst']/tot_i:6.1%} ({a['inst']:.3g})  thr/inst {a['thr']/max(a['inst'],1):5.1f}  "
          + " ".join(f"{n}={v/max(a['samples'],1):.2f}" for v, n in top))
