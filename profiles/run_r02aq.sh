# r02aq: final build (fp64 heavy pieces back to 32: 64 broke the one-entry-per-lane piece load, r02ap)
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu > gpurun_out/r02aq_gpu.log 2>&1; tail -3 gpurun_out/r02aq_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02aq_smoke.txt 2>&1; tail -1 gpurun_out/r02aq_smoke.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/r02aq_bench.json 2> gpurun_out/r02aq_bench.err; tail -c 200 gpurun_out/r02aq_bench.json
