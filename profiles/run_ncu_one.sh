#!/bin/bash
# one --set full capture of kernel $1 (regex) from the small bench; tag $2
K=$1; TAG=${2:-x}; SKIP=${3:-20}
CMD="python bench.py --steps 1 --warmup 3 --roots 256 --e2e-steps 0 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
    -o gpurun_out/prof_${K}_${TAG} -f $CMD > gpurun_out/ncu_${K}_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${K}_${TAG}.log
