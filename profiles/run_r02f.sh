# r02f: owner register budget / items per thread A/B (fp64 cfg2), the warp-per-row bulk owner, sanitizers
cd $GRAFT_REPO_ROOT
LIBS="var/base.so var/m4p3.so var/u2m4p3.so var/u2m3p3.so" bash profiles/abn.sh > gpurun_out/r02f_abn.txt 2>&1
for i in 1 2; do WV_SGNS_BULK_OWNER=1 BENCH_NO_CLOCKS=1 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 > gpurun_out/r02f_bulkowner_$i.json 2>&1; done
python - <<'PY' >> gpurun_out/r02f_abn.txt
import json
for i in (1, 2):
    d = json.loads(open(f"gpurun_out/r02f_bulkowner_{i}.json").read().strip().splitlines()[-1])
    print("bulk-owner", i, round(d["value"] / 1e6, 2), {k[:12]: round(x["ms"] * 1e3, 1) for k, x in d["roofline"]["kernels"].items()})
PY
bash profiles/sanitize.sh > gpurun_out/r02f_sanitize.txt 2>&1
