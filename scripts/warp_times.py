"""Per-warp exit times of one K1 launch (options(diagnostics=1)): how the batch tail
drains (development aid)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2208_09985_b200 as sg
from paper_2208_09985_b200 import _ffi
pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
batch = sg.synth_packed(3, 0, pairs)
s = sg.Session(sg.AlignerConfig(W=64, O=24), batch)
with sg.options(diagnostics=1):
    s.run(); ms, k1 = s.run()
buf = (C.c_uint64 * (3 * 8192))()
n = _ffi.load().sg_session_warp_times(s._h, buf, 8192)
a = np.frombuffer(buf, dtype=np.uint64)[: 3 * n].reshape(n, 3).astype(np.int64)
t0 = a[:, 0].min(); start = (a[:, 0] - t0) / 1e6; end = (a[:, 1] - t0) / 1e6; sm = a[:, 2]
print(f"K1 {k1:.2f} ms, warps {n}, start spread {start.max():.3f} ms")
q = np.percentile(end, [0, 10, 25, 50, 75, 90, 100])
print("warp exit percentiles (ms):", " ".join(f"{x:.1f}" for x in q))
sm_end = np.array([end[sm == k].max() for k in np.unique(sm)])
sm_w = np.array([(sm == k).sum() for k in np.unique(sm)])
print("SM last-exit percentiles (ms):", " ".join(f"{x:.1f}" for x in np.percentile(sm_end, [0, 10, 50, 90, 100])))
for w in np.unique(sm_w):
    print(f"  SMs with {w} warps: {np.sum(sm_w == w)}, mean last exit {sm_end[sm_w == w].mean():.1f} ms")
# average active warps over time
T = end.max(); ts = np.linspace(0, T, 200)
act = np.array([np.sum((start <= t) & (end > t)) for t in ts])
print("active warps vs time (fraction of peak):", " ".join(f"{x:.2f}" for x in act[::20] / act.max()))
print(f"mean active / peak = {act.mean() / act.max():.3f}")
