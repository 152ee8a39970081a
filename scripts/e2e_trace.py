"""Phase timestamps of the end-to-end call (options(diagnostics=4)), development aid:
e2e_trace.py [pairs] [cfg] [nopipe]."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_09985_b200 as sg
pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
cfg_id = int(sys.argv[2]) if len(sys.argv) > 2 else 3
diag = 4 | (8 if len(sys.argv) > 3 and sys.argv[3] == "nopipe" else 0)
batch = sg.synth_packed(cfg_id, 0, pairs)
cfg = sg.AlignerConfig(W=64, O=24)
for rep in range(4):
    t0 = time.perf_counter()
    with sg.options(diagnostics=diag if rep == 3 else diag & 8):
        r = sg.align_packed(cfg, batch, devices=[0])
    t1 = time.perf_counter()
    print(f"rep {rep}: align_packed {1e3 * (t1 - t0):.2f} ms  (device {r.device_ms:.2f} ms, k1 {r.kernel_ms:.2f} ms, launches {r.gpu_launches})", flush=True)
    del r
