# r02n: GPU suite with the per-precision heavy schedule + the new downstream tests; A/B vs the previous
# build (fp64, fp32); north_star target end to end in fp64
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu > gpurun_out/r02n_gpu.log 2>&1; tail -4 gpurun_out/r02n_gpu.log
LIBS="var/cur.so var/new.so" bash profiles/abn.sh > gpurun_out/r02n_abn64.txt 2>&1
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --precision fp32" LIBS="var/cur.so var/new.so" bash profiles/abn.sh > gpurun_out/r02n_abn32.txt 2>&1
python profiles/northstar_e2e.py 10000000 1048576 fp64 > gpurun_out/northstar_e2e_r02n_fp64.json 2>&1
