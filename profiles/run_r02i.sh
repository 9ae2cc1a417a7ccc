# r02i: gather ring A/B (fp64 + fp32), cfg5 walk kernel ncu capture (DRAM bytes, L2 hit rate, stalls)
cd $GRAFT_REPO_ROOT
LIBS="var/cur.so var/gw12s2.so var/gw6s4.so" bash profiles/abn.sh > gpurun_out/r02i_abn64.txt 2>&1
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --precision fp32" LIBS="var/cur.so var/gw12s2.so var/gw6s4.so" bash profiles/abn.sh > gpurun_out/r02i_abn32.txt 2>&1
OUT=gpurun_out/prof_random_walk_kernel_cfg5_r02i
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:random_walk_kernel -s 1 -c 1 -o $OUT -f python profiles/cfg5_walk_prof.py > $OUT.log 2>&1
ncu -i $OUT.ncu-rep --page details --csv > $OUT.details.csv 2>/dev/null
ncu -i $OUT.ncu-rep --page raw --csv > $OUT.raw.csv 2>/dev/null
gzip -f $OUT.raw.csv; rm -f $OUT.ncu-rep
