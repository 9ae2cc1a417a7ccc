# r02v: re-entry check of the restored build (GPU suite, smoke, headline bench)
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -x > gpurun_out/r02v_gpu.log 2>&1; tail -4 gpurun_out/r02v_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.txt 2>&1; tail -2 gpurun_out/r02v_smoke.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/r02v_bench.json 2> gpurun_out/r02v_bench.err; tail -c 600 gpurun_out/r02v_bench.json
# gather ring width A/B (fp64 wide rows): 5x3 (in-tree) vs 8x2, 9x2, 10x2
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/w8s2.so var/w9s2.so var/w10s2.so" bash profiles/abn.sh > gpurun_out/r02v_abn_ring.txt 2>&1
cat gpurun_out/r02v_abn_ring.txt
