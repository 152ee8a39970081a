"""Per-phase instruction and ALU-pipe instruction counts of K1 from an ncu report
(development aid). Phases by source line ranges of window_align.cu."""
import csv, re, subprocess, sys, os, tempfile
from collections import defaultdict
rep = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
td = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2208_09985_b200/_lib/libscrooge_b200.so")], cwd=td, capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, "window_align.sm_100a.cubin")], capture_output=True, text=True).stdout
sec = "k1_window_alignILi2E"; addr_line, addr_op, cur, inside = {}, {}, None, False
for ln in dis.split("\n"):
    if ".text." in ln and "//---" in ln: inside = sec in ln; continue
    if not inside: continue
    m = re.search(r'line (\d+)', ln)
    if "//## File" in ln and m: cur = int(m.group(1)); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)', ln)
    if m and cur is not None:
        a = int(m.group(1), 16); addr_line[a] = cur; addr_op[a] = m.group(3)
src = open(os.path.join(ROOT, "paper_2208_09985_b200/csrc/window_align.cu")).read().split("\n")
def find(pat):
    return next(i + 1 for i, l in enumerate(src) if pat in l)
marks = [("sweep", find("// ---------------------------------------------------------------- skewed DC sweep")),
         ("kernel", find("// ------------------------------------------------------------------ K1")),
         ("setup", find("// ---- lane state ----")),
         ("TB", find("GenASM-TB (traceback.cpp")),
         ("end", find("template <int L> size_t smem_bytes()"))]
def phase(l):
    if l is None: return "?"
    if l < marks[0][1]: return "util"
    if l < marks[1][1]: return "DC"
    if l < marks[2][1]: return "main"
    if l < marks[3][1]:
        if "dc_chunk" in src[l-1] or "DC chunks" in src[l-1]: return "DC"
        return "setup/main"
    if l < marks[4][1]: return "TB"
    return "other"
ALU = {"LOP3", "SHF", "IADD3", "ISETP", "SEL", "LEA", "PRMT", "FLO", "BREV", "POPC", "VIADD", "IMNMX", "VIMNMX", "VIMNMX3", "VIADDMNMX", "PLOP3", "IABS", "BMSK", "LOP"}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.split("\n")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
H = rows[hdr]; ix = {k: H.index(k) for k in H}
data = [r for r in rows[hdr + 1:] if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
agg = defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
for r in data:
    a = int(r[0], 16) - base; p = phase(addr_line.get(a)); op = addr_op.get(a, "?")
    ex = float(r[ix["Instructions Executed"]] or 0)
    g = agg[p]; g[0] += ex; g[1] += ex if op in ALU else 0; g[2] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    g[3] += float(r[ix["Thread Instructions Executed"]] or 0)
ti = sum(g[0] for g in agg.values()); ta = sum(g[1] for g in agg.values()); ts = sum(g[2] for g in agg.values())
print(f"total inst {ti:.3g}  ALU inst {ta:.3g}")
for p, g in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    print(f"{p:11s} samples {g[2]/ts:6.1%}  inst {g[0]:.3g} ({g[0]/ti:5.1%})  ALU {g[1]:.3g} ({g[1]/ta:5.1%})  thr/inst {g[3]/max(g[0],1):4.1f}")
