# r02an: compute-sanitizer memcheck / racecheck / synccheck on the final build (concurrent single-row tiles,
# 10x2 gather ring, high-priority heavy stream)
cd $GRAFT_REPO_ROOT
for T in memcheck racecheck synccheck; do
  timeout 1100 compute-sanitizer --tool $T --kernel-name kns=wv:: --print-limit 50 \
      python profiles/sanitize_workload.py > gpurun_out/sanitize_${T}_r02an.txt 2>&1
  echo "$T exit $?" >> gpurun_out/sanitize_${T}_r02an.txt
  tail -3 gpurun_out/sanitize_${T}_r02an.txt
done
