# r02g: correctness of the split owner (full GPU suite) + A/B of split variants (fp64 cfg2) + timeline
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -x > gpurun_out/r02g_gpu.log 2>&1
tail -3 gpurun_out/r02g_gpu.log
LIBS="var/base.so var/split1.so var/split2.so var/split3.so var/split2m4p3.so" bash profiles/abn.sh > gpurun_out/r02g_abn.txt 2>&1
python profiles/timeline.py fp64 > gpurun_out/timeline_r02g_fp64.txt 2>&1
