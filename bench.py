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


def kernel_source_sha():
    import hashlib
    h = hashlib.sha256()
    for f in ("window_align.cu", "window_align.cuh"):
        with open(os.path.join(ROOT, "paper_2208_09985_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def traffic_bytes(pairs):
    """DRAM bytes (read + write) of one K1 launch, from the committed ncu --set full
    capture of the same workload (profiles/k1_traffic.json). None unless that capture
    was taken of this kernel source (its sha) and this batch size: a stale figure is
    not reported."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as f:
            t = json.load(f)
        if f"{pairs} pairs" not in t["workload"] or t.get("kernel_source_sha") != kernel_source_sha():
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


# ---------------------------------------------------------------- per-config sweep

# Every BASELINE.json config, each measured like the headline (SURVEY §8(d),
# BASELINE.md §4): name, generator id, W, O, pairs, the CPU reference's rate per
# core for sizing its bounded sample, description.
CONFIGS = [
    ("cfg1", 1, 64, 24, 10_000, 17000, "short plumbing: 110/100 bp, 5% edits 1:1:1", (1, 1, 1)),
    ("cfg2", 2, 64, 24, 1_000_000, 9600, "Illumina-like: 250 bp reads, 2% edits 8:1:1", (1, 1, 1)),
    ("cfg4_W32_O12", 4, 32, 12, 20_000, 240, "W/O sweep: 10 kbp, 10% edits 1:1:1", (1, 1, 1)),
    ("cfg4_W64_O24", 4, 64, 24, 20_000, 182, "W/O sweep: 10 kbp, 10% edits 1:1:1", (1, 1, 1)),
    ("cfg4_W64_O33", 4, 64, 33, 20_000, 166, "W/O sweep: 10 kbp, 10% edits 1:1:1", (1, 1, 1)),
    ("cfg4_W128_O48", 4, 128, 48, 20_000, 110, "W/O sweep: 10 kbp, 10% edits 1:1:1", (1, 1, 1)),
    # the early-termination ablation (proj/src/dp.cpp:177, acceptance.cpp:160-194):
    # the same pairs with ET off compute all W + 1 rows of every window
    ("cfg4_W64_O24_et_off", 4, 64, 24, 20_000, 57, "W/O sweep: 10 kbp, 10% edits 1:1:1",
     (1, 1, 0)),
    ("cfg5", 5, 64, 24, 500_000, 300, "mixed 100..20k bp (log-uniform), 30% unrelated", (1, 1, 1)),
]


def digest_name(name, cfg_id, W_, O_, switches):
    s_, d_, e_ = switches
    return f"cfg4_W{W_}_O{O_}_s{s_}d{d_}e{e_}" if cfg_id == 4 else f"cfg{cfg_id}"


def digest_parity(res, name):
    """Every pair of a whole config against the reference's digests
    (tests/golden/digests/<name>.tsv, make_digests.py): blocks bit-exact / total."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import golden_io as G
        import oracle_ffi as Orc
        blocks, pairs, total, _ = G.read_digests(name + ".tsv")
        if pairs != res.n:
            return None
        got, tot = Orc.results_digests(res)
        ok = sum(g == b[2] for g, b in zip(got, blocks))
        return {"blocks_ok": ok, "blocks": len(blocks), "pairs": pairs,
                "all_pairs_bit_exact": ok == len(blocks) and tot == total}
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


def ref_sample(cfg_id, W_, O_, count, threads, switches=(1, 1, 1)):
    tool = ref_tool_path()
    if tool is None:
        return None
    s_, d_, e_ = switches
    out = subprocess.run([tool, "bench", "--cfg", str(cfg_id), "--count", str(count),
                          "--threads", str(threads), "--W", str(W_), "--O", str(O_),
                          "--sene", str(s_), "--dent", str(d_), "--et", str(e_)],
                         capture_output=True, text=True, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def measure_config(sg, name, cfg_id, W_, O_, pairs, rate_per_core, desc, steps, warmup, peak_ops,
                   cpu, switches=(1, 1, 1)):
    s_, d_, e_ = switches
    cfg = sg.AlignerConfig(W=W_, O=O_, sene=bool(s_), dent=bool(d_), early_termination=bool(e_))
    t_gen = time.perf_counter()
    batch = sg.synth_packed(cfg_id, 0, pairs)
    t_gen = time.perf_counter() - t_gen
    sess = sg.Session(cfg, batch, 0)
    for _ in range(warmup):
        sess.run()
    dev, k1 = [], []
    for _ in range(steps):
        ms, k = sess.run()
        dev.append(ms)
        k1.append(k)
    info = sess.info()
    res = sess.fetch()
    sess.close()
    cells = int(res.total.cells_computed)
    alg_ops = 4 * ((W_ + 31) // 32) * cells
    k1_s = sum(k1) / len(k1) / 1e3
    parity = digest_parity(res, digest_name(name, cfg_id, W_, O_, switches))
    launches = int(res.gpu_launches)
    rows = int(res.total.rows_computed)
    del res
    sg.align_packed(cfg, batch)  # warm the one-shot path
    t0 = time.perf_counter()
    for _ in range(steps):
        r = sg.align_packed(cfg, batch)
        del r
    e2e_s = (time.perf_counter() - t0) / steps
    h2d, d2h = sg.last_transfer_bytes()
    out = {
        "workload": f"{name}: {pairs:,} pairs, {desc}, W={W_} O={O_}, "
                    f"sene={s_} dent={d_} et={e_}",
        "value": round(pairs / (sum(dev) / len(dev) / 1e3), 1), "unit": UNIT,
        "ms_per_step": round(sum(dev) / len(dev), 3),
        "e2e": {"value": round(pairs / e2e_s, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "kernel": info["kernel"],
        "roofline": {"bound": "int_alu", "achieved": round(alg_ops / k1_s / 1e12, 3),
                     "peak": round(peak_ops / 1e12, 3), "unit": "Tops/s (int32 lane-ops)",
                     "frac": round(alg_ops / k1_s / peak_ops, 4), "alg_ops_per_launch": alg_ops,
                     "k1_ms": round(1e3 * k1_s, 3)},
        "reference_counters": {"rows_computed": rows, "cells_computed": cells},
        "gpu_launches_per_step": launches,
        "parity": parity,
        "gen_seconds": round(t_gen, 2),
    }
    if cpu:
        threads = os.cpu_count() or 1
        n = int(min(pairs, max(200, rate_per_core * threads * 3)))
        try:
            r = ref_sample(cfg_id, W_, O_, n, threads, switches)
            if r is not None:
                out["cpu_baseline"] = {
                    "value": round(r["pairs_per_second"], 3), "unit": UNIT, "cores": threads,
                    "kind": "reference",
                    "sample": f"first {n:,} {name} pairs, {r['align_seconds']:.2f} s of run_batch"}
                out["speedup_e2e_vs_cpu"] = round(out["e2e"]["value"] / r["pairs_per_second"], 1)
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"error": str(e)}
    return out


# ---------------------------------------------------------------- our arm

def main_ours(args):
    ws, rank, local = dist_env()
    import paper_2208_09985_b200 as sg
    from paper_2208_09985_b200 import _ffi
    L = _ffi.load()
    visible = L.sg_device_count()
    if visible < 1:
        raise SystemExit("bench.py: no CUDA device (the GPU path has no CPU fallback)")
    # N GPUs: one rank per GPU under torchrun, else N devices driven from this process
    inproc = ws == 1
    n_gpus = ws if ws > 1 else args.gpus
    if inproc and visible < n_gpus:
        raise SystemExit(f"bench.py: --gpus {n_gpus} but only {visible} CUDA device(s) visible")
    devices = list(range(n_gpus)) if inproc else [local]
    dist = Dist(ws, rank, local, args.backend)
    pairs = args.pairs
    cfg = sg.AlignerConfig(W=W, O=O, sene=True, dent=True, early_termination=True)

    from paper_2208_09985_b200 import shard
    t_gen = time.perf_counter()
    if inproc:  # device d aligns pairs [d*P, (d+1)*P) of the generator (weak scaling)
        batches = [sg.synth_packed(CFG_ID, d * pairs, pairs) for d in devices]
    else:
        first, count = shard.rank_range(rank, ws, pairs)
        batches = [sg.synth_packed(CFG_ID, first, count)]
    t_gen = time.perf_counter() - t_gen
    sessions = [sg.Session(cfg, b, d) for b, d in zip(batches, devices)]

    # ---- device-resident: value. Each device's steps run on its own host thread;
    # the job time is the max over devices (and ranks) of the summed CUDA-event times.
    def run_steps(k, n_steps, out=None, barrier=None):
        if barrier is not None:
            barrier.wait()
        for _ in range(n_steps):
            ms, k1 = sessions[k].run()
            if out is not None:
                out[k].append((ms, k1))

    def on_all(n_steps, out=None):
        if len(sessions) == 1:
            run_steps(0, n_steps, out)
            return
        bar = threading.Barrier(len(sessions))
        th = [threading.Thread(target=run_steps, args=(k, n_steps, out, bar))
              for k in range(len(sessions))]
        for t in th:
            t.start()
        for t in th:
            t.join()

    on_all(args.warmup)
    info = sessions[0].info()
    sampler = ClockSampler(devices[0])
    sampler.start()
    dist.barrier()
    cuda_sync()
    times = [[] for _ in sessions]
    t0 = time.perf_counter()
    on_all(args.steps, times)
    cuda_sync()
    dist.barrier()
    wall = time.perf_counter() - t0
    clocks = sampler.stop()
    total_ms = dist.max(max(sum(ms for ms, _ in t) for t in times))
    value = n_gpus * pairs * args.steps / (total_ms / 1e3)
    k1_ms = [k1 for ms, k1 in times[0]]

    res = sessions[0].fetch()
    launches_per_step = int(res.gpu_launches) * len(sessions)
    cells = int(res.total.cells_computed)
    alg_ops = 4 * ((W + 31) // 32) * cells
    k1_avg_s = sum(k1_ms) / len(k1_ms) / 1e3
    achieved = alg_ops / k1_avg_s

    # parity: every pair of device 0's batch (rank 0 at N=1 holds cfg3's 100k pairs)
    # against the reference's whole-config digests
    parity = None
    if rank == 0 and pairs == 100000 and (inproc or ws == 1):
        parity = digest_parity(res, "cfg3")
    for s_ in sessions:
        s_.close()
    del res

    # ---- measured ALU peak (roofline denominator)
    import ctypes as C
    r_alu, mhz_peak, ops_s = C.c_double(), C.c_double(), C.c_double()
    L.sg_alu_peak(devices[0], C.byref(r_alu), C.byref(mhz_peak), C.byref(ops_s))
    sm_mhz = clocks["sm_mhz"] if clocks else mhz_peak.value
    peak = info["sms"] * r_alu.value * sm_mhz * 1e6

    # ---- end to end through the C ABI with host buffers: e2e. In one process the
    # library splits one batch of N x P pairs over the N devices itself (K5).
    if inproc and n_gpus > 1:
        e2e_batch = sg.synth_packed(CFG_ID, 0, n_gpus * pairs)
    else:
        e2e_batch = batches[0]
    e2e_devices = devices
    for _ in range(max(1, args.warmup // 2)):
        sg.align_packed(cfg, e2e_batch, devices=e2e_devices)
    dist.barrier()
    cuda_sync()
    t0 = time.perf_counter()
    h2d = d2h = 0
    for _ in range(args.steps):
        r = sg.align_packed(cfg, e2e_batch, devices=e2e_devices)
        h2d, d2h = sg.last_transfer_bytes()
        del r
    cuda_sync()
    dist.barrier()
    e2e_s = dist.max(time.perf_counter() - t0)
    e2e = n_gpus * pairs * args.steps / e2e_s

    base = None
    if rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        try:
            base = cpu_baseline(os.cpu_count() or 1)
        except Exception as e:  # pragma: no cover
            base = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                    "sample": f"failed: {e}"}

    # ---- every other BASELINE config (N = 1, rank 0): BASELINE.md §4's table
    per_config = None
    if rank == 0 and n_gpus == 1 and not args.headline_only:
        del batches, e2e_batch
        per_config = {}
        for (name, cid, w_, o_, n_, rate, desc, sw) in CONFIGS:
            per_config[name] = measure_config(sg, name, cid, w_, o_, n_, rate, desc,
                                              args.config_steps, args.warmup, peak,
                                              not args.no_cpu_baseline, sw)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": n_gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32 bitvectors (int)",
            "data": "synthetic (seeded cfg3 generator)",
            "config": {"workload": WORKLOAD, "pairs_per_gpu": pairs, "W": W, "O": O,
                       "parallelism": (f"{n_gpus} GPU(s) driven from one process, "
                                       "pairs sharded, no collective") if inproc else
                                      f"one rank per GPU ({ws}), pairs sharded, no collective",
                       "l2": "inputs 0.5 GB/GPU > 126 MB L2, no flush needed",
                       "resident_lanes": info["lanes"], "kernel": info["kernel"]},
            "roofline": {"bound": "int_alu", "achieved": round(achieved / 1e12, 3),
                         "peak": round(peak / 1e12, 3), "unit": "Tops/s (int32 lane-ops)",
                         "frac": round(achieved / peak, 4), "traffic": traffic_bytes(pairs),
                         "traffic_unit": "DRAM bytes per K1 launch (ncu --set full of this "
                                         "kernel build, profiles/k1_traffic.json)",
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
            "configs": per_config,
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
    ap.add_argument("--headline-only", action="store_true",
                    help="skip the per-config sweep (cfg1, cfg2, cfg4 x 4, cfg5) at N = 1")
    ap.add_argument("--config-steps", type=int, default=3, help="timed steps per config")
    args = ap.parse_args()
    if args.impl == "reference":
        return main_reference(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
