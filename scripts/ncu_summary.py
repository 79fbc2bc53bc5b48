#!/usr/bin/env python
"""Summarise an ncu --set full report (and optionally a launch-list CSV) into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_c2.ncu-rep profiles/r01_c2_v1 \
        [--launches gpurun_out/launches.csv] [--config c2] [--flops F]

Writes <out>.txt (human-readable) and <out>.json (the numbers bench.py's roofline
``traffic`` field and DESIGN.md cite).  Runs here (no GPU): it only reads the report.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__sass_inst_executed_op_shared_ld.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers",
    "sm__cycles_elapsed.avg.per_second",
]

TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TO_NS = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    return [(dict(zip(head, r)), dict(zip(head, units))) for r in rows[2:]]


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def summarise(rep: str, flops: float | None):
    res = []
    for d, u in raw_rows(rep):
        e = {"kernel": d.get("Kernel Name"), "metrics": {}}
        for m in METRICS:
            if m in d:
                e["metrics"][m] = {"value": num(d[m]), "unit": u.get(m, "")}
        stalls = {k.split("issue_stalled_")[1].split("_per_issue")[0]: num(v)
                  for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        e["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))[:10])
        m = e["metrics"]
        rb = m.get("dram__bytes_read.sum")
        wb = m.get("dram__bytes_write.sum")
        if rb and wb:
            e["dram_bytes_per_launch"] = rb["value"] * TO_BYTES.get(rb["unit"], 1) + \
                wb["value"] * TO_BYTES.get(wb["unit"], 1)
        t = m.get("gpu__time_duration.sum")
        if t:
            e["time_ns"] = t["value"] * TO_NS.get(t["unit"], 1)
            if flops:
                e["tflops_under_ncu"] = flops / e["time_ns"] / 1e3
        res.append(e)
    return res


def executed_fmas(rep: str):
    """Thread-level FMAs the kernel executed, from the SASS source page: every FFMA
    counts 1 per thread, every packed FFMA2 2 (SURVEY.md §8(d) FFMA efficiency =
    useful FMAs / executed FMAs).  Also the share of warp-stall samples on the FFMA /
    FFMA2 instructions."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next((r for r in rows if "Source" in r and "Thread Instructions Executed" in r), None)
    if hdr is None:
        return None
    i_src, i_thr = hdr.index("Source"), hdr.index("Thread Instructions Executed")
    i_smp = hdr.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in hdr else None
    fma = 0.0
    smp_all = smp_fma = 0.0
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= i_thr:
            continue
        op = r[i_src].split()
        if not op:
            continue
        opc = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        n = num(r[i_thr]) or 0.0
        smp = num(r[i_smp]) or 0.0 if i_smp is not None else 0.0
        smp_all += smp
        if opc.startswith("FFMA2"):
            fma += 2 * n
            smp_fma += smp
        elif opc.startswith("FFMA"):
            fma += n
            smp_fma += smp
    return {"executed_fmas": fma, "ffma_stall_sample_share": smp_fma / smp_all if smp_all else None}


def launches(path: str):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r["Metric Unit"]))
    agg = {}
    for k, v, unit in rows:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v * TO_NS.get(unit, 1)
    total = sum(a[1] for a in agg.values()) or 1.0
    return {k: {"launches": a[0], "mean_ns": a[1] / a[0], "share": a[1] / total} for k, a in agg.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--config", default="")
    ap.add_argument("--flops", type=float)
    ap.add_argument("--traffic-json", help="merge {config: {kernel, dram_bytes_per_launch}} into this file")
    ap.add_argument("--kernel-name", default="pipe", help="library kernel name recorded with the traffic")
    a = ap.parse_args()
    s = {"report": a.report, "config": a.config, "kernels": summarise(a.report, a.flops)}
    if a.flops:
        ex = executed_fmas(a.report)
        if ex and ex["executed_fmas"]:
            ex["useful_fmas"] = a.flops / 2
            ex["ffma_efficiency"] = ex["useful_fmas"] / ex["executed_fmas"]
            s["ffma"] = ex
    if a.launches:
        s["launch_list"] = launches(a.launches)
    with open(a.out + ".json", "w") as f:
        json.dump(s, f, indent=1)
    with open(a.out + ".txt", "w") as f:
        f.write(f"ncu --set full summary of {a.report} (config {a.config})\n")
        for e in s["kernels"]:
            f.write(f"\nkernel: {e['kernel']}\n")
            for k, v in e["metrics"].items():
                f.write(f"  {k:70s} {v['value']} {v['unit']}\n")
            if "dram_bytes_per_launch" in e:
                f.write(f"  {'dram read+write bytes per launch':70s} {e['dram_bytes_per_launch']:.0f}\n")
            if "tflops_under_ncu" in e:
                f.write(f"  {'useful TFLOP/s under ncu (serialised, cold)':70s} {e['tflops_under_ncu']:.2f}\n")
            f.write("  top stall reasons (warps per issue-active cycle):\n")
            for k, v in e["stalls_per_issue"].items():
                f.write(f"    {k:40s} {v}\n")
        if "ffma" in s:
            x = s["ffma"]
            f.write(f"\nFFMA efficiency (useful FMAs / executed thread FMAs, FFMA2 = 2): "
                    f"{x['useful_fmas']:.4g} / {x['executed_fmas']:.4g} = {x['ffma_efficiency']:.3f}\n")
        if "launch_list" in s:
            f.write("\nlaunch list (ncu gpu__time_duration.sum, --clock-control none):\n")
            for k, v in s["launch_list"].items():
                f.write(f"  {v['launches']:4d} x {v['mean_ns'] / 1e3:9.2f} us  share {v['share']:.3f}  {k}\n")
    print(open(a.out + ".txt").read())
    if a.traffic_json and s["kernels"] and "dram_bytes_per_launch" in s["kernels"][0]:
        try:
            with open(a.traffic_json) as f:
                t = json.load(f)
        except (OSError, ValueError):
            t = {}
        t[a.config] = {"kernel": a.kernel_name,
                       "dram_bytes_per_launch": int(s["kernels"][0]["dram_bytes_per_launch"]),
                       "source": os.path.basename(a.out) + ".txt"}
        with open(a.traffic_json, "w") as f:
            json.dump(t, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    sys.exit(main())
