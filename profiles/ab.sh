#!/bin/bash
# A/B on one box: A = default build/env, B = $BLIB (library path) and/or $BENV ("VAR=val ...")
ARGS=${ARGS:-"--steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline"}
BCMD="env ${BENV:-} ${BLIB:+WV_LIB=$BLIB}"
for i in 1 2; do
  python bench.py $ARGS > gpurun_out/abA$i.json 2> gpurun_out/abA$i.err
  $BCMD python bench.py $ARGS > gpurun_out/abB$i.json 2> gpurun_out/abB$i.err
done
python - <<'PY'
import json
for v in "AB":
    for i in (1, 2):
        try:
            d = json.load(open(f"gpurun_out/ab{v}{i}.json"))
            r = d["roofline"]["kernels"]
            print(v, i, round(d["value"] / 1e6, 2), "Mpairs/s", {k[:12]: round(x["ms"] * 1e3, 1) for k, x in r.items()})
        except Exception as e:
            print(v, i, "ERR", e, open(f"gpurun_out/ab{v}{i}.err").read()[-500:])
PY
