#!/usr/bin/env python3
"""Summarise ncu captures (run here, on reports fetched from the GPU box).

  python scripts/ncu_summary.py --rep gpurun_out/prof.ncu-rep --key cfg3/tree/t1048576 \
      --launches gpurun_out/launches.csv --out profiles/r1_ncu_cfg3_p1.md

Writes a markdown summary (per-kernel duration, DRAM bytes, throughput,
registers, tensor-pipe activity, stall breakdown) and merges
{key: {"dram_bytes_per_launch": ...}} for the split kernel into
profiles/ncu_summary.json, which bench.py reads for roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]
UNIT_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--key", required=True, help="workload/algo/t<shard tokens>, e.g. cfg3/tree/t1048576 (bench.py looks traffic up by it)")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    hdr, units, rows = raw(args.rep)
    lines = [f"# ncu summary: {args.key}", "", args.note, "",
             f"Source: `{os.path.basename(args.rep)}` (`ncu --set full --clock-control none`, cold-cache replay: "
             "compare shares, not absolute times, with the bench's CUDA-event numbers).", ""]
    split_bytes = None
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        lines.append(f"## `{name[:90]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        vals = {}
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"| {label} (`{m}`) | {r[i]} | {units[i]} |")
                vals[m] = (r[i], units[i])
        if name.startswith("void k1_") or name.startswith("k1_"):
            try:
                rb = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * UNIT_SCALE.get(vals["dram__bytes_read.sum"][1], 1)
                wb = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * UNIT_SCALE.get(vals["dram__bytes_write.sum"][1], 1)
                split_bytes = rb + wb
                us = float(vals["gpu__time_duration.sum"][0].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(
                    vals["gpu__time_duration.sum"][1], 1.0)
                lines.append(f"| kernel-only DRAM read rate (read bytes / duration) | {rb / (us * 1e-6) / 1e9:.1f} | GB/s |")
            except (KeyError, ValueError):
                pass
        lines.append("")
    # stall reasons of the split kernel (source-level totals)
    src = subprocess.run(["ncu", "-i", args.rep, "--page", "details", "--section", "WarpStateStats", "--csv"],
                         capture_output=True, text=True).stdout
    if src:
        lines += ["## Warp state statistics (all captured kernels)", "", "```", src.strip()[:4000], "```", ""]
    if args.launches and os.path.exists(args.launches):
        lines += ["## Launch list (`--metrics gpu__time_duration.sum`)", "", "| kernel | duration | unit |", "|---|---|---|"]
        with open(args.launches) as f:
            txt = [ln for ln in f if not ln.startswith("==")]
        lrows = list(csv.reader(txt))
        h = None
        for lr in lrows:
            if lr and lr[0] == "ID":
                h = lr
                continue
            if h and len(lr) == len(h):
                d = dict(zip(h, lr))
                lines.append(f"| {d['Kernel Name'][:70]} | {d['Metric Value']} | {d['Metric Unit']} |")
        lines.append("")
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if split_bytes is not None:
        path = os.path.join(os.path.dirname(args.out), "ncu_summary.json")
        data = json.load(open(path)) if os.path.exists(path) else {}
        data[args.key] = {"dram_bytes_per_launch": split_bytes, "report": os.path.basename(args.rep)}
        with open(path, "w") as f:
            json.dump(data, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
