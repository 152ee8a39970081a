"""K6 (wide windows) throughput probe on seeded synthetic pairs (development aid).

    python scripts/wide_perf.py CFG COUNT W O [reps]
Prints device ms (K6 + K2/K3, CUDA events) and alignments/s for a Session run.
"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_09985_b200 as sg
cfg_id, count, W, Ov = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
b = sg.synth_packed(cfg_id, 0, count)
s = sg.Session(sg.AlignerConfig(W=W, O=Ov), b)
for r in range(reps):
    ms, k1 = s.run()
    print(f"cfg{cfg_id} n={count} W={W} O={Ov}: device {ms:.2f} ms, kernel {k1:.2f} ms, "
          f"{count / (ms / 1e3):.0f} aln/s")
