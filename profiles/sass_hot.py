#!/usr/bin/env python
"""Summarise an exported ncu SASS source page (gpurun_out/prof_*.sass.csv.gz): total
executed warp instructions, stall samples, and the hottest instructions/opcode mix."""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(gzip.open(path, "rt")))
hdr = rows[1]
iA, iS, iW, iN, iE = (hdr.index(x) for x in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                               "Warp Stall Sampling (Not-issued Samples)", "Instructions Executed"))
data = []
for r in rows[2:]:
    try:
        data.append((r[iA], r[iS].strip(), int(r[iW] or 0), int(r[iN] or 0), int(r[iE] or 0)))
    except (ValueError, IndexError):
        pass
tot_e = sum(d[4] for d in data)
tot_s = sum(d[2] for d in data)
print(f"{rows[0][1]}\n executed warp instructions {tot_e:,}; stall samples {tot_s:,}")
ops = collections.Counter()
for d in data:
    ops[d[1].split()[0] if not d[1].startswith("@") else d[1].split()[1]] += d[4]
print(" opcode mix:", ", ".join(f"{k} {v / tot_e:.1%}" for k, v in ops.most_common(14)))
print(" hottest (stall samples):")
for d in sorted(data, key=lambda x: -x[2])[:top]:
    print(f"  {d[0][-5:]} {d[2]:6d} {d[3]:6d} {d[4]:9d}  {d[1][:90]}")
