#!/bin/bash
# Round evidence (one B200, under gpurun).  Part "bench": default bench line,
# reference arm, ncu launch list of a small bench.  Part "ncu": --set full
# captures of the main kernels (kept under gpurun's 64 MiB copy-back limit).
TAG=${1:-r01}; PART=${2:-bench}
CMD="python bench.py --steps 1 --warmup 3 --roots 256 --e2e-steps 0 --no-cpu-baseline"
# .ncu-rep files are too large for gpurun's 64 MiB copy-back: keep CSV pages
# (details, raw metrics, SASS source with per-line stalls) and drop the report
export_rep() {
  ncu -i $1.ncu-rep --page details --csv > $1.details.csv 2>/dev/null
  ncu -i $1.ncu-rep --page raw --csv > $1.raw.csv 2>/dev/null
  ncu -i $1.ncu-rep --page source --csv --print-source sass > $1.sass.csv 2>/dev/null
  gzip -f $1.raw.csv $1.sass.csv
  rm -f $1.ncu-rep
}
if [ "$PART" = bench ]; then
  python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
  python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_list_${TAG}.log 2>&1
  gzip -f gpurun_out/launches_${TAG}.csv
else
  for K in sgns_owner_flat heavy_piece_kernel heavy_order group_order sgns_gather_bulk sgns_decode group_segments group_place_rank; do
    ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
        -o gpurun_out/prof_${K}_${TAG} -f $CMD > gpurun_out/ncu_${K}_${TAG}.log 2>&1
    export_rep gpurun_out/prof_${K}_${TAG}
  done
  # the walk kernel at the bench's own block size (8192 roots -> 819,200 walkers)
  ncu --set full --clock-control none --import-source on -k regex:random_walk_kernel -s 1 -c 1 \
      -o gpurun_out/prof_random_walk_kernel_${TAG} -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 \
      --no-cpu-baseline > gpurun_out/ncu_random_walk_kernel_${TAG}.log 2>&1
  export_rep gpurun_out/prof_random_walk_kernel_${TAG}
fi
