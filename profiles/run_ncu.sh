#!/bin/bash
# ncu evidence for bench.py (run under gpurun on one B200; outputs land in gpurun_out/).
#   1. launch list (device time per launch; cold-cache & serialised -> compare shares)
#   2. --set full captures of the SGNS owner/Adam, SGNS pair and walk kernels
# The bench is run with a small root block (--roots 256) so ncu's per-launch
# replay stays tractable; kernel shapes per batch are identical to the default
# run (the batch size comes from the reference's 1 GiB rule either way).
set -u
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 3 --roots 256 --e2e-steps 0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_list_${TAG}.log 2>&1
for K in sgns_owner_kernel sgns_pair_kernel random_walk_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 2 \
      -o gpurun_out/prof_${K}_${TAG} -f $CMD > gpurun_out/ncu_${K}_${TAG}.log 2>&1
done
