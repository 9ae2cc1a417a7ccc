# r02ap: fp64 heavy pieces of 64 contributions: GPU suite, smoke, headline bench
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu > gpurun_out/r02ap_gpu.log 2>&1; tail -3 gpurun_out/r02ap_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ap_smoke.txt 2>&1; tail -1 gpurun_out/r02ap_smoke.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/r02ap_bench.json 2> gpurun_out/r02ap_bench.err; tail -c 300 gpurun_out/r02ap_bench.json
