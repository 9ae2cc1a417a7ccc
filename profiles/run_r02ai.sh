# r02ai: ncu of the real cfg2 step (full 8192-root block, not the 256-root launch-list workload):
# --set full of the gather and the single-row tiles, and a 450-launch list from inside the first step
cd $GRAFT_REPO_ROOT
export BENCH_ARGS="--roots 8192"
for K in sgns_gather_bulk_kernel sgns_owner_single_kernel heavy_piece_kernel; do
  CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --roots 8192"
  OUT=gpurun_out/prof_${K}_r02ai_full
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 300 -c 1 -o $OUT -f $CMD > $OUT.log 2>&1
  ncu -i $OUT.ncu-rep --page details --csv > $OUT.details.csv 2>/dev/null
  ncu -i $OUT.ncu-rep --page raw --csv > $OUT.raw.csv 2>/dev/null
  gzip -f $OUT.raw.csv; rm -f $OUT.ncu-rep
done
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3000 -c 450 --csv --log-file gpurun_out/launches_r02ai_full.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 > gpurun_out/r02ai_launch_bench.log 2>&1
gzip -f gpurun_out/launches_r02ai_full.csv
python profiles/ncu_brief.py gpurun_out/prof_*_r02ai_full.details.csv
