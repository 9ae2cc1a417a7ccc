# r02q: the headline bench line (default flags) and its wall time
cd $GRAFT_REPO_ROOT
s=$(date +%s); python bench.py > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err; e=$(date +%s)
echo "bench wall s: $((e - s))" >> gpurun_out/r02q_bench.err
