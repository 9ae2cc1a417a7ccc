# r02s: the lean single-contribution owner -- parity (SGNS suites), A/B vs without (WV_NO_SINGLES) and
# with 64 registers (sing4), fp64 and fp32
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_sgns.py tests/test_gpu_sgns_shapes.py tests/test_shard_gpu.py tests/test_dist_gpu.py -q -x > gpurun_out/r02s_tests.log 2>&1; tail -3 gpurun_out/r02s_tests.log
for P in fp64 fp32; do
  A="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --precision $P"
  for i in 1 2; do
    BENCH_NO_CLOCKS=1 WV_LIB=var/sing5.so python bench.py $A > gpurun_out/ab_sing5_${P}_$i.json 2>/dev/null
    BENCH_NO_CLOCKS=1 WV_NO_SINGLES=1 WV_LIB=var/sing5.so python bench.py $A > gpurun_out/ab_nosing_${P}_$i.json 2>/dev/null
    BENCH_NO_CLOCKS=1 WV_LIB=var/sing4.so python bench.py $A > gpurun_out/ab_sing4_${P}_$i.json 2>/dev/null
  done
done
python - <<'PY' > gpurun_out/r02s_ab.txt
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], round(d["value"] / 1e6, 2), {k[:12]: round(x["ms"] * 1e3, 1) for k, x in d["roofline"]["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
