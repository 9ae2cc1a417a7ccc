# r02k: evidence set -- GPU suite, smoke, full bench (fp64 headline + extras), reference arm,
# ncu launch list of a short bench, ncu --set full of the update / gather / walk kernels
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu > gpurun_out/r02k_gpu.log 2>&1; tail -3 gpurun_out/r02k_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k_smoke.txt 2>&1; tail -2 gpurun_out/r02k_smoke.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02k_bench_ref.json 2> gpurun_out/r02k_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r02k.csv python bench.py --steps 1 --warmup 3 --roots 256 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 > gpurun_out/r02k_launch_bench.log 2>&1
gzip -f gpurun_out/launches_r02k.csv
for K in sgns_owner_flat_kernel sgns_gather_bulk_kernel heavy_piece_kernel random_walk_kernel; do
  timeout 600 bash profiles/ncu_one.sh $K r02k
done
python profiles/timeline.py fp64 > gpurun_out/timeline_r02k_fp64.txt 2>&1
python profiles/cfg5_walks.py > gpurun_out/r02k_cfg5_walks.json 2>&1
