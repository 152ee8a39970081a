"""When each warp of the mixed K1 last had work (options(diagnostics=1)): the end of the
batch by role (7 band + 2 cooperative warps per block). Development aid.
usage: warp_last_busy.py [cfg] [pairs] [W] [O]"""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2208_09985_b200 as sg
from paper_2208_09985_b200 import _ffi
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
W = int(sys.argv[3]) if len(sys.argv) > 3 else 64; O = int(sys.argv[4]) if len(sys.argv) > 4 else 24
batch = sg.synth_packed(cfg, 0, n)
s = sg.Session(sg.AlignerConfig(W=W, O=O), batch)
with sg.options(diagnostics=1):
    s.run(); ms, k1 = s.run()
buf = (C.c_uint64 * (3 * 8192))()
cnt = _ffi.load().sg_session_warp_times(s._h, buf, 8192)
a = np.frombuffer(buf, dtype=np.uint64)[: 3 * cnt].reshape(cnt, 3).astype(np.int64)
idx = np.arange(cnt); wib = idx % 9
ok = a[:, 0] > 0
t0 = a[ok, 0].min()
end = (a[:, 1] - t0) / 1e6
print("K1", k1, "warps", ok.sum())
for name, sel in (("band", (wib < 7) & ok), ("coop", (wib >= 7) & ok)):
    e = end[sel]
    if len(e): print(name, len(e), "last-busy percentiles (ms):", " ".join(f"{x:.1f}" for x in np.percentile(e, [0, 10, 50, 90, 99, 100])))
