"""Top source lines of K1<L> in an ncu report (stall samples), via nvdisasm line info.
usage: ncu_lines.py <report.ncu-rep> [L] [N]  (development aid)"""
import csv, re, subprocess, sys, os, tempfile
from collections import defaultdict
rep = sys.argv[1]; L = sys.argv[2] if len(sys.argv) > 2 else "2"; N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
td = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2208_09985_b200/_lib/libscrooge_b200.so")], cwd=td, capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, "window_align.sm_100a.cubin")], capture_output=True, text=True).stdout
sec = os.environ.get("SG_SEC", f"k1_window_alignILi{L}E")
addr_line, cur, inside = {}, None, False
for ln in dis.split("\n"):
    if ".text." in ln and "//---" in ln:
        inside = sec in ln; continue
    if not inside: continue
    m = re.search(r'line (\d+)', ln)
    if "//## File" in ln and m: cur = int(m.group(1)); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur is not None: addr_line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.split("\n")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
H = rows[hdr]; ix = {k: H.index(k) for k in H}
data = [r for r in rows[hdr + 1:] if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
agg = defaultdict(lambda: [0.0, 0.0, 0.0]); st = defaultdict(lambda: defaultdict(float))
stall_cols = [k for k in H if k.startswith("stall_") and "Not Issued" not in k]
for r in data:
    l = addr_line.get(int(r[0], 16) - base)
    a = agg[l]; a[0] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    a[1] += float(r[ix["Instructions Executed"]] or 0); a[2] += float(r[ix["Thread Instructions Executed"]] or 0)
    for k in stall_cols: st[l][k] += float(r[ix[k]] or 0)
tot = sum(a[0] for a in agg.values()); toti = sum(a[1] for a in agg.values())
src = open(os.path.join(ROOT, "paper_2208_09985_b200/csrc/window_align.cu")).read().split("\n")
print(f"total samples {tot:.0f} instructions {toti:.3g}")
for l, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    top = sorted(((v, k[6:]) for k, v in st[l].items()), reverse=True)[:2]
    print(f"{l}: {a[0]/tot:6.1%} inst {a[1]/toti:5.1%} thr {a[2]/max(a[1],1):4.1f} {[t[1] for t in top]} | {src[l-1].strip()[:80] if l else ''}")
