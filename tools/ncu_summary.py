"""Summarise ncu reports / launch lists into profiles/ (committed evidence).

    python tools/ncu_summary.py --rep gpurun_out/prof_k2_r01.ncu-rep [--rep ...] \
        --launches gpurun_out/launches_r01.csv --out profiles/r01_ncu_summary.md
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.sum", "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_lg_throttle",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
        res.append(d)
    return res


def launches(path):
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    total = 0.0
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6,
                 "second": 1e3, "s": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        per[name][0] += 1
        per[name][1] += v * scale
        total += v * scale
    return per, total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        per, total = launches(a.launches)
        lines += ["## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
                  "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (n, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {n} | {ms:.3f} | {ms / total:.3f} |")
        lines.append(f"| total | {sum(v[0] for v in per.values())} | {total:.3f} | 1.000 |")
        lines.append("")
    for rep in a.rep:
        for d in raw(rep):
            lines += [f"## `{d['kernel'][:110]}`", f"source: `{rep.split('/')[-1]}` (ncu --set full)", "",
                      "| metric | value | unit |", "|---|---|---|"]
            for k in KEYS:
                if k in d:
                    lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
            lines.append("")
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
