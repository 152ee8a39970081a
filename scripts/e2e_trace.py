"""Phase timestamps of the end-to-end call (options(diagnostics=4)), development aid."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_09985_b200 as sg
pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
batch = sg.synth_packed(3, 0, pairs)
cfg = sg.AlignerConfig(W=64, O=24)
for rep in range(3):
    t0 = time.perf_counter()
    with sg.options(diagnostics=4):
        r = sg.align_packed(cfg, batch, devices=[0])
    t1 = time.perf_counter()
    print(f"rep {rep}: align_packed {1e3 * (t1 - t0):.2f} ms  (device {r.device_ms:.2f} ms, k1 {r.kernel_ms:.2f} ms)", flush=True)
    t2 = time.perf_counter(); del r; print(f"  free {1e3 * (time.perf_counter() - t2):.2f} ms", flush=True)
