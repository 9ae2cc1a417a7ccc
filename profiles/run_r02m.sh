# r02m: heavy pieces serial before the light rows (light rows then own the SMs), fp64 and fp32
cd $GRAFT_REPO_ROOT
LIBS="var/cur.so var/ser4.so var/ser4b.so var/ser5.so" bash profiles/abn.sh > gpurun_out/r02m_abn64.txt 2>&1
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --precision fp32" LIBS="var/cur.so var/ser4.so var/ser4b.so var/ser5.so" bash profiles/abn.sh > gpurun_out/r02m_abn32.txt 2>&1
