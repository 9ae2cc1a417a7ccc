# r02r: heavy pieces -- unrolled partial reduction (pu4), 16-contribution fp64 pieces (p16); fp64 + fp32;
# fp64 replay parity at the cfg2 shape (the heavy-row reassociation changes with the piece size)
cd $GRAFT_REPO_ROOT
LIBS="var/base.so var/pu4.so var/p16.so" bash profiles/abn.sh > gpurun_out/r02r_abn64.txt 2>&1
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --precision fp32" LIBS="var/base.so var/pu4.so" bash profiles/abn.sh > gpurun_out/r02r_abn32.txt 2>&1
WV_LIB=var/p16.so python -m pytest tests/test_gpu_sgns_shapes.py tests/test_gpu_sgns.py -q -x > gpurun_out/r02r_p16_tests.log 2>&1; tail -2 gpurun_out/r02r_p16_tests.log
