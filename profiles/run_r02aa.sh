# r02aa: single-contribution rows concurrent with the heavy pieces + multi-contribution rows (short-lived tiles)
cd $GRAFT_REPO_ROOT
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/cc4.so var/cc8.so var/cc2.so var/cc4lo.so" bash profiles/abn.sh > gpurun_out/r02aa_abn.txt 2>&1
cat gpurun_out/r02aa_abn.txt
WV_LIB=var/cc4.so python profiles/timeline.py fp64 > gpurun_out/timeline_r02aa_cc4_fp64.txt 2>&1; tail -2 gpurun_out/timeline_r02aa_cc4_fp64.txt
WV_LIB=var/cc4.so timeout 900 python -m pytest tests/test_gpu_sgns_shapes.py tests/test_gpu_sgns.py -q -x 2>&1 | tail -3
