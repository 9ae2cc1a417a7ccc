# r02ah: fp32 store with the single-contribution rows split out and run concurrently (tiles of 12 / 24)
cd $GRAFT_REPO_ROOT
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --precision fp32" LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/f1.so var/f1t24.so" bash profiles/abn.sh > gpurun_out/r02ah_abn.txt 2>&1
cat gpurun_out/r02ah_abn.txt
