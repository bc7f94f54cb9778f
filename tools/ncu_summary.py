"""Summarise ncu artefacts for profiles/: launch list shares + key metrics of full captures.

python tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep ... > profiles/x.md
"""

from __future__ import annotations

import argparse
import collections
import csv
import subprocess
import sys

KEEP = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Executed Instructions",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:48]
            tot[name] += float(r[vi].replace(",", ""))
            cnt[name] += 1
    grand = sum(tot.values())
    out = ["| kernel | launches | total ms | avg ms | share |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:14]:
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / cnt[k] / 1e6:.3f} | {v / grand * 100:.1f}% |")
    return "\n".join(out)


def rep(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    h = rows[0]
    ni, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    name = rows[1][ni].split("(")[0]
    out = [f"**{name}**", "", "| metric | value |", "|---|---|"]
    seen = set()
    for r in rows[1:]:
        if r[mi] in KEEP and r[mi] not in seen:
            seen.add(r[mi])
            out.append(f"| {r[mi]} | {r[vi]} {r[ui]} |")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        hh, units, vals = rr[0], rr[1], rr[2]
        for key in RAW:
            if key in hh:
                i = hh.index(key)
                out.append(f"| `{key}` | {vals[i]} {units[i]} |")
        stalls = []
        for i, n in enumerate(hh):
            if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
                try:
                    stalls.append((float(vals[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = ", ".join(f"{n} {s / tot * 100:.0f}%" for s, n in sorted(stalls)[::-1][:5])
        out.append(f"| top stall reasons (pc sampling) | {top} |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    a = ap.parse_args()
    if a.launches:
        print("### Launch list (ncu --metrics gpu__time_duration.sum, cold-cache serialised)\n")
        print(launches(a.launches))
        print()
    for r in a.rep:
        print(rep(r))
        print()


if __name__ == "__main__":
    sys.exit(main())
