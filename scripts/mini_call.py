"""One small one-shot call (development aid, e.g. under compute-sanitizer):
mini_call.py [pairs] [cfg] [diagnostics bits] [kernel]."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_09985_b200 as sg
pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
cfg_id = int(sys.argv[2]) if len(sys.argv) > 2 else 1
diag = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kernel = sys.argv[4] if len(sys.argv) > 4 else "auto"
batch = sg.synth_packed(cfg_id, 0, pairs)
with sg.options(diagnostics=diag, kernel=kernel):
    r = sg.align_packed(sg.AlignerConfig(W=64, O=24), batch, devices=[0])
print("ok", int(r.distance[:pairs].sum()), r.gpu_launches, f"{r.device_ms:.3f} ms")
