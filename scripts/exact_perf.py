"""K7 (exact global alignment) throughput probe on seeded synthetic pairs (development aid).

    python scripts/exact_perf.py CFG COUNT [budget_bytes]
"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_09985_b200 as sg
cfg_id, count = int(sys.argv[1]), int(sys.argv[2])
budget = int(sys.argv[3]) if len(sys.argv) > 3 else None
b = sg.synth_packed(cfg_id, 0, count)
for r in range(2):
    t0 = time.perf_counter()
    with sg.options(exact_budget=budget):
        res = sg.global_align_packed(b)
    t1 = time.perf_counter()
    print(f"cfg{cfg_id} n={count}: device {res.device_ms:.1f} ms (K7 {res.kernel_ms:.1f} ms, "
          f"{int(res.gpu_launches)} launches), wall {1e3 * (t1 - t0):.1f} ms, "
          f"{count / (res.device_ms / 1e3):.0f} pairs/s")
