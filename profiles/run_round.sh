#!/bin/bash
# Round evidence (one B200, under gpurun).  Part "bench": default bench line,
# reference arm, ncu launch list of a small bench.  Part "ncu": --set full
# captures of the main kernels (kept under gpurun's 64 MiB copy-back limit).
TAG=${1:-r01}; PART=${2:-bench}
CMD="python bench.py --steps 1 --warmup 3 --roots 256 --e2e-steps 0 --no-cpu-baseline"
if [ "$PART" = bench ]; then
  python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
  python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_list_${TAG}.log 2>&1
  gzip -f gpurun_out/launches_${TAG}.csv
else
  for K in sgns_owner_kernel sgns_heavy_kernel sgns_gather_bulk sgns_decode; do
    ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
        -o gpurun_out/prof_${K}_${TAG} -f $CMD > gpurun_out/ncu_${K}_${TAG}.log 2>&1
  done
  ncu --set full --clock-control none --import-source on -k regex:random_walk_kernel -s 1 -c 1 \
      -o gpurun_out/prof_random_walk_kernel_${TAG} -f $CMD > gpurun_out/ncu_random_walk_kernel_${TAG}.log 2>&1
fi
