# r02j: walk adjacency (one load per hop) -- parity + cfg5 walk rate with and without it; GPU suite; full bench
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -x > gpurun_out/r02j_gpu.log 2>&1
tail -3 gpurun_out/r02j_gpu.log
python profiles/cfg5_walks.py > gpurun_out/r02j_cfg5_adj.json 2>&1
WV_NO_WALK_ADJ=1 python profiles/cfg5_walks.py > gpurun_out/r02j_cfg5_csr.json 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
