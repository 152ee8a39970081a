#!/usr/bin/env python
"""Benchmark: windowed GenASM alignments/s on N B200s (BASELINE.json metric).

Workload (one "step" = one pass of the hot path over one batch):
  BASELINE cfg3, the headline long-read config: 100,000 pairs per GPU of
  10 kbp reads (text = read + 5% slack), 15% edits sub:ins:del = 2:5:3,
  W=64, O=24, SENE + DENT + early termination on. Seeded synthetic pairs
  (paper_2208_09985_b200/csrc/synth.c, seed 3; rank r aligns pairs
  [r*100000, (r+1)*100000) of the generator: weak scaling, no collective on
  the data path). Packed inputs are 0.5 GB per GPU (> the 126 MB L2), so no
  L2 flush is needed between steps.

value  = alignments/s with inputs already in HBM (K1 + K2 + K3 per step,
         CUDA events on the library's stream, max over ranks).
e2e    = alignments/s through the C ABI with HOST buffers (sg_align_packed:
         pinned H2D of the packed pairs, kernels, D2H of distances, windows,
         counters and CIGAR run bytes), wall clock, max over ranks.
roofline = K1's ALG_OPS (4 * ceil(W/32) * cells_computed, SURVEY.md §8(d),
         from the per-pair counters that match the reference) / K1 time,
         against the measured integer-ALU peak of the box.
cpu_baseline = the unmodified reference run_batch (oracle/_ref/ref_tool) on
         this host's cores, bounded sample, rank 0 at N=1.

--impl reference times the reference CPU aligner alone (same JSON keys).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG_ID = 3
W, O = 64, 24
WORKLOAD = ("cfg3 long noisy reads: 100,000 pairs/GPU x 10 kbp (text +5% slack), 15% edits "
            "2:5:3, W=64 O=24, SENE+DENT+ET")
METRIC = "alignments/sec"
UNIT = "alignments/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Dist:
    """Barrier + max-over-ranks through torch.distributed (plumbing only)."""

    def __init__(self, ws, rank, local, backend):
        self.ws, self.rank = ws, rank
        self.torch = None
        if ws > 1:
            import torch
            import torch.distributed as td
            self.torch, self.td = torch, td
            if backend == "nccl":
                torch.cuda.set_device(local)
            td.init_process_group(backend=backend)
            self.dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")

    def barrier(self):
        if self.torch is not None:
            self.td.barrier()

    def max(self, v: float) -> float:
        if self.torch is None:
            return v
        t = self.torch.tensor([float(v)], dtype=self.torch.float64, device=self.dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.torch is not None:
            self.td.destroy_process_group()


def cuda_sync():
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
    except Exception:
        pass


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(
            ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
             "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
            stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------- reference arm

def ref_tool_path():
    p = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    return p if os.path.exists(p) else None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference_sample(pairs: int, threads: int, first: int = 0):
    """The unmodified reference run_batch on a bounded cfg3 sample (rank 0)."""
    tool = ref_tool_path()
    if tool is None:
        return None
    out = subprocess.run([tool, "bench", "--cfg", str(CFG_ID), "--first", str(first),
                          "--count", str(pairs), "--threads", str(threads), "--W", str(W),
                          "--O", str(O)], capture_output=True, text=True, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def run_port_sample(pairs: int, threads: int):
    """Fallback when oracle/_ref is absent: the C restatement (oracle/), threaded."""
    from concurrent.futures import ThreadPoolExecutor
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as Orc
    spec = Orc.baseline_spec(CFG_ID)
    data = [Orc.synth_pair(spec, k) for k in range(pairs)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda tp: Orc.align(tp[0], tp[1], W=W, O=O), data))
    dt = time.perf_counter() - t0
    return {"pairs": pairs, "threads": threads, "align_seconds": dt, "pairs_per_second": pairs / dt}


def reference_sample_size(threads: int) -> int:
    # ~150 cfg3 pairs/s per core for the reference -> ~8-10 s
    return int(min(100000, max(200, threads * 1200)))


def traffic_bytes(pairs):
    """DRAM bytes (read + write) of one K1 launch, from the committed ncu --set full
    capture of the same workload (profiles/k1_traffic.json); None if it does not
    match this run's batch size."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as f:
            t = json.load(f)
        if f"{pairs} pairs" not in t["workload"]:
            return None
        return int(t["dram_bytes_read"]) + int(t["dram_bytes_write"])
    except (OSError, KeyError, ValueError):
        return None


def cpu_baseline(threads: int):
    n = reference_sample_size(threads)
    r = run_reference_sample(n, threads)
    kind = "reference"
    if r is None:
        n = max(64, n // 8)
        r = run_port_sample(n, threads)
        kind = "port"
    return {"value": round(r["pairs_per_second"], 3), "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"first {n} cfg3 pairs, {r['align_seconds']:.2f} s of run_batch "
                      f"(alignment only, batch.cpp:83-92) on {cpu_model()}"}


def main_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = reference_sample_size(threads)
    times, kind = [], "reference"
    for step in range(args.warmup + args.steps):
        r = run_reference_sample(n, threads)
        if r is None:
            kind = "port"
            n = max(64, n // 8)
            r = run_port_sample(n, threads)
        if step >= args.warmup:
            times.append(r["align_seconds"])
    value = n * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 bitvectors", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_pairs_per_step": n, "W": W, "O": O},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"first {n} cfg3 pairs per step on {cpu_model()}"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm

def main_ours(args):
    ws, rank, local = dist_env()
    dist = Dist(ws, rank, local, args.backend)
    import paper_2208_09985_b200 as sg
    from paper_2208_09985_b200 import _ffi
    L = _ffi.load()
    if L.sg_device_count() < 1:
        raise SystemExit("bench.py: no CUDA device (the GPU path has no CPU fallback)")
    device = local if ws > 1 else 0
    pairs = args.pairs
    cfg = sg.AlignerConfig(W=W, O=O, sene=True, dent=True, early_termination=True)

    from paper_2208_09985_b200 import shard
    first, count = shard.rank_range(rank, ws, pairs)
    t_gen = time.perf_counter()
    batch = sg.synth_packed(CFG_ID, first, count)
    t_gen = time.perf_counter() - t_gen
    sess = sg.Session(cfg, batch, device)

    # ---- device-resident: value
    for _ in range(args.warmup):
        sess.run()
    info = sess.info()
    sampler = ClockSampler(device)
    sampler.start()
    dist.barrier()
    cuda_sync()
    dev_ms, k1_ms = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ms, k1 = sess.run()
        dev_ms.append(ms)
        k1_ms.append(k1)
    cuda_sync()
    dist.barrier()
    wall = time.perf_counter() - t0
    clocks = sampler.stop()
    total_ms = dist.max(sum(dev_ms))
    value = ws * pairs * args.steps / (total_ms / 1e3)

    res = sess.fetch()
    launches_per_step = int(res.gpu_launches)
    cells = int(res.total.cells_computed)
    alg_ops = 4 * ((W + 31) // 32) * cells
    k1_avg_s = sum(k1_ms) / len(k1_ms) / 1e3
    achieved = alg_ops / k1_avg_s

    # parity sample against the reference's golden vectors (rank 0 holds pairs 0..)
    parity = None
    if rank == 0:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import golden_io as G
            import oracle_ffi as Orc
            ok = tot = 0
            for name in ("cfg3_head.tsv", "cfg3_tail.tsv"):
                for row in G.read_golden(name):
                    k = G.pair_index(row["id"])
                    if k >= pairs:
                        continue
                    cig = res.cigar_string(k)
                    tot += 1
                    ok += (int(res.distance[k]) == row["distance"] and
                           Orc.fnv1a(cig) == row["hash"] and int(res.windows[k]) == row["windows"]
                           and [int(x) for x in res.counters[k]] == row["counters"])
            parity = f"{ok}/{tot} pairs bit-exact vs reference golden vectors"
        except Exception as e:  # pragma: no cover
            parity = f"unchecked ({e})"
    sess.close()
    del res

    # ---- measured ALU peak (roofline denominator)
    import ctypes as C
    r_alu, mhz_peak, ops_s = C.c_double(), C.c_double(), C.c_double()
    L.sg_alu_peak(device, C.byref(r_alu), C.byref(mhz_peak), C.byref(ops_s))
    sm_mhz = clocks["sm_mhz"] if clocks else mhz_peak.value
    peak = info["sms"] * r_alu.value * sm_mhz * 1e6

    # ---- end to end through the C ABI with host buffers: e2e
    for _ in range(max(1, args.warmup // 2)):
        sg.align_packed(cfg, batch, devices=[device])
    dist.barrier()
    cuda_sync()
    t0 = time.perf_counter()
    h2d = d2h = 0
    for _ in range(args.steps):
        r = sg.align_packed(cfg, batch, devices=[device])
        h2d, d2h = sg.last_transfer_bytes()
        del r
    cuda_sync()
    dist.barrier()
    e2e_s = dist.max(time.perf_counter() - t0)
    e2e = ws * pairs * args.steps / e2e_s

    base = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            base = cpu_baseline(os.cpu_count() or 1)
        except Exception as e:  # pragma: no cover
            base = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                    "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32 bitvectors (int)",
            "data": "synthetic (seeded cfg3 generator)",
            "config": {"workload": WORKLOAD, "pairs_per_gpu": pairs, "W": W, "O": O,
                       "parallelism": f"pairs sharded over {ws} GPU(s), no collective",
                       "l2": "inputs 0.5 GB/GPU > 126 MB L2, no flush needed",
                       "resident_lanes": info["lanes"]},
            "roofline": {"bound": "int_alu", "achieved": round(achieved / 1e12, 3),
                         "peak": round(peak / 1e12, 3), "unit": "Tops/s (int32 lane-ops)",
                         "frac": round(achieved / peak, 4), "traffic": traffic_bytes(pairs),
                         "traffic_unit": "DRAM bytes per K1 launch (ncu, profiles/k1_traffic.json)",
                         "alg_ops_per_launch": alg_ops, "cells_computed": cells,
                         "k1_ms": round(sum(k1_ms) / len(k1_ms), 3),
                         "r_alu_ops_per_clk_per_sm": round(r_alu.value, 2),
                         "peak_basis": f"{info['sms']} SMs x measured LOP3 rate x "
                                       f"{sm_mhz:.0f} MHz (median under load)"},
            "e2e": {"value": round(e2e, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "parity": parity,
            "cpu_baseline": base,
            "host": {"gen_seconds": round(t_gen, 2), "wall_s_timed": round(wall, 3)},
        }
        print(json.dumps(line), flush=True)
    dist.close()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--pairs", type=int, default=100000, help="pairs per GPU (cfg3: 100000)")
    ap.add_argument("--backend", default="nccl", help="torch.distributed backend for N>1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return main_reference(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
