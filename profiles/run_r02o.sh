# r02o: block-wise session quality tests; A/B: segment-record prefetch, 10- and 12-warp gather rings;
# north_star target with one global epoch (fp64)
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_sgns.py -q -k "blockwise or two_clique" > gpurun_out/r02o_tests.log 2>&1; tail -4 gpurun_out/r02o_tests.log
LIBS="var/new.so var/segpf.so var/gw10.so var/gw12s3.so" bash profiles/abn.sh > gpurun_out/r02o_abn64.txt 2>&1
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --precision fp32" LIBS="var/new.so var/segpf.so var/gw10.so var/gw12s3.so" bash profiles/abn.sh > gpurun_out/r02o_abn32.txt 2>&1
python profiles/northstar_e2e.py 10000000 0 fp64 > gpurun_out/northstar_e2e_r02o_fp64.json 2>&1
