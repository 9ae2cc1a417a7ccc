#!/bin/bash
# One ncu --set full capture of kernel regex $1 (20th launch) from a small bench, exported to CSV pages.
#   bash profiles/ncu_one.sh <kernel-regex> <tag>    (WV_LIB selects a library variant)
K=$1; TAG=${2:-x}
CMD="python bench.py --steps 1 --warmup 3 --roots 256 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 ${BENCH_ARGS:-}"
OUT=gpurun_out/prof_${K}_${TAG}
ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 -o $OUT -f $CMD > $OUT.log 2>&1
ncu -i $OUT.ncu-rep --page details --csv > $OUT.details.csv 2>/dev/null
ncu -i $OUT.ncu-rep --page raw --csv > $OUT.raw.csv 2>/dev/null
ncu -i $OUT.ncu-rep --page source --csv --print-source sass > $OUT.sass.csv 2>/dev/null
gzip -f $OUT.raw.csv $OUT.sass.csv
rm -f $OUT.ncu-rep
