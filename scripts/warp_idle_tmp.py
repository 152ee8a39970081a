import ctypes as C, os, sys
os.environ["SG_WARP_TIMES"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2208_09985_b200 as sg
from paper_2208_09985_b200 import _ffi
batch = sg.synth_packed(int(sys.argv[1]) if len(sys.argv) > 1 else 3, 0, int(sys.argv[2]) if len(sys.argv) > 2 else 100000)
W = int(sys.argv[3]) if len(sys.argv) > 3 else 64; O = int(sys.argv[4]) if len(sys.argv) > 4 else 24
s = sg.Session(sg.AlignerConfig(W=W, O=O), batch)
s.run(); ms, k1 = s.run()
lib = _ffi.load()
lib.sg_debug_warp_times.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * (3 * 8192))()
n = lib.sg_debug_warp_times(buf, 8192)
a = np.frombuffer(buf, dtype=np.uint64)[: 3 * n].reshape(n, 3).astype(np.int64); n = int((a[:, 0] > 0).sum()); a = a[:n]
t0 = a[:, 0].min(); end = (a[:, 1] - t0) / 1e6
wib = np.arange(n) % 9
print("K1", k1, "warps", n)
for name, sel in (("band", wib < 7), ("coop", wib >= 7)):
    e = end[sel]
    print(name, "last-busy percentiles (ms):", " ".join(f"{x:.1f}" for x in np.percentile(e, [0, 10, 50, 90, 99, 100])))
fe = a[:, 2][wib < 7]
fe = fe[fe > 0]
if len(fe): print("band fresh-exhausted (ms):", " ".join(f"{x:.1f}" for x in np.percentile(((fe << 20) - t0) / 1e6, [0, 50, 100])))
