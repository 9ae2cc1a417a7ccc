# r02c: fp64 row-traffic microbenchmark, ncu --set full captures of the fp64 SGNS kernels,
# launch list of a short fp64 bench, and the new multi-rank device tests
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rows64 profiles/micro/rows64_bench.cu && /tmp/rows64 > gpurun_out/r02c_rows64.txt 2>&1
python -m pytest tests/test_dist_gpu.py tests/test_shard_gpu.py -q -x > gpurun_out/r02c_dist_tests.log 2>&1
for K in sgns_owner_flat_kernel sgns_gather_bulk_kernel heavy_piece_kernel sgns_decode_kernel; do
  timeout 600 bash profiles/ncu_one.sh $K r02c
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r02c.csv python bench.py --steps 1 --warmup 3 --roots 256 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 > gpurun_out/r02c_launch_bench.log 2>&1
gzip -f gpurun_out/launches_r02c.csv
