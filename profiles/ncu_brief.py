#!/usr/bin/env python
"""Print the key ncu --set full metrics of exported reports (gpurun_out/prof_*.details.csv)."""
import csv
import sys
from pathlib import Path

KEEP = {
    "GPU Speed Of Light Throughput": ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
                                      "L1/TEX Cache Throughput", "Compute (SM) Throughput"],
    "Memory Workload Analysis": ["Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate"],
    "Occupancy": ["Achieved Occupancy", "Theoretical Occupancy", "Block Limit Registers", "Block Limit Shared Mem"],
    "Launch Statistics": ["Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block"],
    "Scheduler Statistics": ["Issued Warp Per Scheduler", "No Eligible"],
    "Warp State Statistics": ["Warp Cycles Per Issued Instruction"],
}


def brief(path: Path) -> list[str]:
    rows = list(csv.reader(open(path)))
    h = rows[0]
    iS, iN, iV, iU = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Value", "Metric Unit"))
    out = []
    for r in rows[1:]:
        if r[iS] in KEEP and r[iN] in KEEP[r[iS]]:
            out.append(f"{r[iN]} {r[iV]} {r[iU]}".strip())
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(Path(p).name.replace(".details.csv", ""), "::", "; ".join(brief(Path(p))))
