"""Summarize ncu captures into the committed profiles/ directory.

    python tools/ncu_summary.py --round r1 --launches gpurun_out/launches_r1.csv \
        --reports gpurun_out/r1_filter.ncu-rep gpurun_out/r1_others.ncu-rep

Writes profiles/<round>_launches.md (per-kernel device-time shares from the
cold-cache, serialised launch list) and profiles/<round>_kernels.json /
profiles/<round>_kernels.md (per-launch DRAM traffic, throughput, occupancy
from --set full captures).  Needs the ncu CLI (present in this image).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def short(name):
    n = name.split("(")[0]
    return n.split("::")[-1]


def launches(path):
    """Per kernel: launch times (s) and DRAM bytes, from an ncu --csv metrics list."""
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, ni, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    ii = hdr.index("ID")
    per = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9 if "time" in r[ni] else 1.0)
        per.setdefault((r[ii], short(r[ki])), {})[r[ni]] = v
    agg = collections.OrderedDict()
    for (_, k), m in per.items():
        a = agg.setdefault(k, {"t": [], "rd": 0.0, "wr": 0.0})
        a["t"].append(m.get("gpu__time_duration.sum", 0.0))
        a["rd"] += m.get("dram__bytes_read.sum", 0.0)
        a["wr"] += m.get("dram__bytes_write.sum", 0.0)
    return agg


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, k in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    d[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    d[k] = None
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r1")
    ap.add_argument("--launches")
    ap.add_argument("--reports", nargs="*", default=[])
    ap.add_argument("--name", default="launches", help="output file suffix for the launch list")
    ap.add_argument("--command", default="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.launches:
        agg = launches(a.launches)
        tot = sum(sum(v["t"]) for v in agg.values())
        lines = [f"# {a.round}: kernel launch list (ncu gpu__time_duration + DRAM bytes, --clock-control none)", "",
                 f"Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 f"--clock-control none --csv {a.command}` (cold-cache and serialised: compare shares, not "
                 "absolutes).", "",
                 "| kernel | launches | total ms | mean ms | share | DRAM read MB | DRAM write MB |",
                 "|---|---|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]["t"])):
            t = v["t"]
            lines.append(f"| {k} | {len(t)} | {sum(t) * 1e3:.3f} | {sum(t) / len(t) * 1e3:.4f} | "
                         f"{sum(t) / tot:.3f} | {v['rd'] / 1e6:.1f} | {v['wr'] / 1e6:.1f} |")
        open(os.path.join(ROOT, "profiles", f"{a.round}_{a.name}.md"), "w").write("\n".join(lines) + "\n")
    kern = []
    for p in a.reports:
        kern += report(p)
    if kern:
        json.dump(kern, open(os.path.join(ROOT, "profiles", f"{a.round}_kernels.json"), "w"), indent=1)
        lines = [f"# {a.round}: ncu --set full captures (per launch)", "",
                 "| kernel | time ms | DRAM read MB | DRAM write MB | DRAM % peak | SM % | warps active % | "
                 "FP64 pipe % | DMMA pipe % | regs | grid x block |", "|---|---|---|---|---|---|---|---|---|---|---|"]
        for d in kern:
            g = lambda k, s=1.0, f="{:.2f}": (f.format(d[k] * s) if d.get(k) is not None else "-")
            lines.append(f"| {d['kernel']} | {g('time', 1e3, '{:.3f}')} | {g('dram_read', 1e-6, '{:.1f}')} | "
                         f"{g('dram_write', 1e-6, '{:.1f}')} | {g('dram_pct')} | {g('sm_pct')} | "
                         f"{g('warps_active_pct')} | {g('fp64_pipe_pct')} | {g('dmma_pipe_pct')} | "
                         f"{g('regs', 1, '{:.0f}')} | "
                         f"{g('grid', 1, '{:.0f}')} x {g('block', 1, '{:.0f}')} |")
        open(os.path.join(ROOT, "profiles", f"{a.round}_kernels.md"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
