"""Summarise ncu evidence into profiles/ (run here, no GPU needed).

python tools/ncu_summary.py --rep gpurun_out/X.ncu-rep [--launches gpurun_out/launches.csv]
                            --out profiles/NAME.md [--cells N]
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess
from collections import defaultdict

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "SM Frequency"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Scheduler Statistics", "Active Warps Per Scheduler"),
    ("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    ("Scheduler Statistics", "No Eligible"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Warp State Statistics", "Avg. Active Threads Per Warp"),
    ("Instruction Statistics", "Executed Instructions"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Block Size"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Occupancy", "Achieved Active Warps Per SM"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
]
RAW = [
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def details(rep: str) -> list[tuple[str, str]]:
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))))
    hdr = rows[0]
    out = {}
    name = ""
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", name)
        out[(d.get("Section Name"), d.get("Metric Name"))] = f"{d.get('Metric Value')} {d.get('Metric Unit')}"
    return name, [(m, out.get((s, m), "-")) for s, m in KEYS]


def raw(rep: str) -> list[tuple[str, str]]:
    text = ncu("-i", rep, "--page", "raw")
    got = {}
    for line in text.splitlines():
        parts = line.split()
        if len(parts) >= 2 and parts[0] in RAW:
            got[parts[0]] = " ".join(parts[1:])
    return [(k, got.get(k, "-")) for k in RAW]


def hotspots(rep: str, top: int = 15) -> list[str]:
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source",
                                           "cuda,sass"))))
    hdr = rows[2]
    H = len(hdr)
    idx = {h: i - H for i, h in enumerate(hdr)}

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0

    lines, ti, ts = [], 0, 0
    for r in rows[3:]:
        if not r or r[0] == "" or len(r) < H:
            continue
        ie = num(r[idx["Instructions Executed"]])
        sm = num(r[idx["Warp Stall Sampling (All Samples)"]])
        src = ",".join(r[1:len(r) - H + 2]).strip()[:88]
        lines.append((r[0], src, ie, sm))
        ti += ie
        ts += sm
    out = [f"| line | instr % | stall-sample % | source |", "|---|---|---|---|"]
    for ln, src, ie, sm in sorted(lines, key=lambda x: -x[2])[:top]:
        out.append(f"| {ln} | {100 * ie / max(ti, 1):.1f} | {100 * sm / max(ts, 1):.1f} | `{src}` |")
    return out


def launches(path: str) -> list[str]:
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            ns = v * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
                      "second": 1e9, "s": 1e9}.get(unit, 1)
            agg[d["Kernel Name"][:90]][0] += 1
            agg[d["Kernel Name"][:90]][1] += ns
    tot = sum(v[1] for v in agg.values())
    out = ["| launches | total ms | share | kernel |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
        out.append(f"| {c} | {t / 1e6:.3f} | {100 * t / tot:.2f}% | `{k}` |")
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    name, det = details(args.rep)
    md = [f"# {args.title}", "", args.note, "", f"Kernel: `{name}`", "", "| metric | value |",
          "|---|---|"]
    md += [f"| {k} | {v} |" for k, v in det]
    md += [f"| {k} | {v} |" for k, v in raw(args.rep)]
    md += ["", "## Source hotspots (instructions executed, stall samples)", ""] + hotspots(args.rep)
    if args.launches:
        md += ["", "## Launch list (ncu gpu__time_duration, cold-cache, serialised)", ""]
        md += launches(args.launches)
    with open(args.out, "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
