# $TAG: final evidence set for the current build
TAG=${1:-r02t}
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu > gpurun_out/${TAG}_gpu.log 2>&1; tail -4 gpurun_out/${TAG}_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -2 gpurun_out/${TAG}_smoke.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/${TAG}_bench_2rank_gloo.json 2> gpurun_out/${TAG}_bench_2rank_gloo.err
# launch list: 450 launches from inside the first step of the real cfg2 workload (8192-root block)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3000 -c 450 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 > gpurun_out/${TAG}_launch_bench.log 2>&1
gzip -f gpurun_out/launches_$TAG.csv
export BENCH_ARGS="--roots 8192"
for K in sgns_owner_single_kernel sgns_owner_flat_kernel sgns_gather_bulk_kernel heavy_piece_kernel; do timeout 600 bash profiles/ncu_one.sh $K $TAG; done
python profiles/timeline.py fp64 > gpurun_out/timeline_${TAG}_fp64.txt 2>&1
