#!/bin/bash
# --set full captures of the SGNS kernels at steady state of the DEFAULT bench
# workload (8192-root blocks; skip the first 9000 launches of each kernel).
TAG=${1:-r01}; SKIP=${2:-9000}
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
for K in ${KERNELS:-sgns_owner_bulk sgns_heavy sgns_gather_bulk sgns_decode group_place group_segments}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
      -o gpurun_out/steady_${K}_${TAG} -f $CMD > gpurun_out/ncu_steady_${K}_${TAG}.log 2>&1
  tail -1 gpurun_out/ncu_steady_${K}_${TAG}.log
done
