#!/bin/bash
# A/B/n on one box: one short bench per library variant (WV_LIB), twice each.
#   LIBS="path1 path2 ..." bash profiles/abn.sh
ARGS=${ARGS:-"--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0"}
for i in 1 2; do
  for L in $LIBS; do
    n=$(basename $L .so)
    BENCH_NO_CLOCKS=1 WV_LIB=$L python bench.py $ARGS > gpurun_out/abn_${n}_$i.json 2> gpurun_out/abn_${n}_$i.err
  done
done
python - "$LIBS" <<'PY'
import json, sys, os
for L in sys.argv[1].split():
    n = os.path.basename(L)[:-3]
    for i in (1, 2):
        try:
            d = json.load(open(f"gpurun_out/abn_{n}_{i}.json"))
            r = d["roofline"]["kernels"]
            print(f"{n:28s} {i} {d['value'] / 1e6:7.2f} Mpairs/s", {k[:12]: round(x["ms"] * 1e3, 1) for k, x in r.items()})
        except Exception as e:
            print(n, i, "ERR", e, open(f"gpurun_out/abn_{n}_{i}.err").read()[-300:])
PY
