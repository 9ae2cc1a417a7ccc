#!/usr/bin/env python
"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
kernels captured with ncu --set full (gpurun_out/prof_<kernel>_<tag>.raw.csv.gz)
-> profiles/traffic_<tag>.json, which bench.py reports as roofline.traffic."""
import csv
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {}
for p in sorted((ROOT / "gpurun_out").glob(f"prof_*_{tag}.raw.csv.gz")):
    rows = list(csv.reader(gzip.open(p, "rt")))
    hdr, units, val = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, v, u in zip(hdr, val, units)}
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = d[m]
        b += float(v.replace(",", "")) * UNIT.get(u, 1)
    k = p.name[len("prof_"):-len(f"_{tag}.raw.csv.gz")]
    out[k] = {"dram_bytes": b, "duration_us": float(d["gpu__time_duration.sum"][0].replace(",", "")) *
              (1e-3 if d["gpu__time_duration.sum"][1] == "nsecond" else 1.0),
              "l2_hit_rate_pct": float(d["lts__t_sector_hit_rate.pct"][0].replace(",", ""))
              if "lts__t_sector_hit_rate.pct" in d else None,
              "kernel": d["Kernel Name"][0][:120]}
(ROOT / "profiles" / f"traffic_{tag}.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
