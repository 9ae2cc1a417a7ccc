#!/bin/bash
# compute-sanitizer over profiles/sanitize_workload.py (SURVEY §5 race detection): memcheck,
# racecheck (shared-memory hazards), synccheck and initcheck on the library's kernels only
# (--kernel-name kns=wv::).  Summaries -> gpurun_out/sanitize_<tool>.txt
cd ${GRAFT_REPO_ROOT:-.}
for T in memcheck racecheck synccheck initcheck; do
  X=""; [ "$T" = initcheck ] && X="--check-api-memory-access no"  # host copies of torch-initialised scalars are not instrumented
  timeout 1500 compute-sanitizer --tool $T $X --kernel-name kns=wv:: --print-limit 50 \
      python profiles/sanitize_workload.py > gpurun_out/sanitize_$T.txt 2>&1
  echo "$T exit $?" >> gpurun_out/sanitize_$T.txt
  tail -3 gpurun_out/sanitize_$T.txt
done
