"""Summarise the per-config ncu metric CSVs of scripts/gpu/ncu_configs.sh into a
markdown table (development aid): per K1 launch its time, DRAM bytes and GB/s,
shared-memory pipe %, issue %, ALU / FMA pipe %, warp instructions."""
import csv, glob, os, re, sys

def load(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                  "Metric Unit", "ID"))
    launches = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"kernel": r[ki]})
        v = r[vi].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            pass
        d[r[mi]] = (v, r[ui])
    return list(launches.values())

def val(d, k, unit_to=None):
    v, u = d.get(k, (float("nan"), ""))
    if unit_to == "ms":
        return v / 1e6 if u == "ns" else v / 1e3 if u == "us" else v
    if unit_to == "MB":
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
        return v * scale
    return v

def main(tag, out):
    lines = ["| config | kernel | time ms | DRAM read MB | DRAM write MB | DRAM GB/s (r+w) | smem pipe % | issue % | ALU % | FMA % | warp inst (M) | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for path in sorted(glob.glob(f"gpurun_out/{tag}_ncu_cfg*.csv")):
        cfg = re.search(r"ncu_(cfg\d+_W\d+_O\d+)", path).group(1)
        for d in load(path):
            name = re.sub(r"\(.*", "", d["kernel"]).replace("void ", "").replace("unnamed>::", "")
            t = val(d, "gpu__time_duration.sum", "ms")
            rd = val(d, "dram__bytes_read.sum", "MB")
            wr = val(d, "dram__bytes_write.sum", "MB")
            gbs = (rd + wr) / t if t else float("nan")
            lines.append(f"| {cfg} | {name} | {t:.3f} | {rd:.1f} | {wr:.1f} | {gbs:.0f} | "
                         f"{val(d, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed'):.1f} | "
                         f"{val(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                         f"{val(d, 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
                         f"{val(d, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
                         f"{val(d, 'sm__inst_executed.sum') / 1e6:.0f} | "
                         f"{val(d, 'launch__registers_per_thread'):.0f} |")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
