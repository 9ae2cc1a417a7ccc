#!/usr/bin/env python
"""DRAM traffic per launch of the SGNS batch kernels, averaged over
every launch in an ncu launch list (profiles/r02/launches_<tag>.csv.gz, metrics
gpu__time_duration.sum + dram__bytes_read.sum + dram__bytes_write.sum; cold caches,
serialised) -> profiles/traffic_<tag>.json, which bench.py reports as roofline.traffic.

    python profiles/traffic_from_launches.py r02p
"""
import collections
import csv
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KERNELS = ("sgns_decode_kernel", "group_segments", "group_place_rank", "group_order", "heavy_order",
           "sgns_gather_bulk_kernel", "sgns_owner_flat_kernel", "sgns_owner_single_kernel", "heavy_piece_kernel")

tag = sys.argv[1]
path = ROOT / "profiles" / "r02" / f"launches_{tag}.csv.gz"
rows = list(csv.reader(gzip.open(path, "rt")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
iK, iM, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(lambda: collections.defaultdict(dict))
for r in rows[hi + 1:]:
    name = r[iK].split("(")[0].split("<")[0].replace("void ", "").replace("wv::", "")
    if name not in KERNELS:
        continue
    try:
        per[name][r[iID]][r[iM]] = float(r[iV].replace(",", ""))
    except ValueError:
        continue
out = {}
for name, launches in per.items():
    ls = list(launches.values())
    b = [x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0) for x in ls]
    t = [x.get("gpu__time_duration.sum", 0.0) for x in ls]
    out[name] = {"dram_bytes": sum(b) / len(b), "duration_us": sum(t) / len(t) / 1e3, "launches": len(ls),
                 "source": f"profiles/r02/launches_{tag}.csv.gz (ncu launch list, cold caches, serialised)"}
(ROOT / "profiles" / f"traffic_{tag}.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
