# r02ak: next batch's grouping after the gather (decode still beside it); fp64 fallback-ring parity test
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sgns_shapes.py -q -k fallback 2>&1 | tail -3
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/sg2.so" bash profiles/abn.sh > gpurun_out/r02ak_abn.txt 2>&1
cat gpurun_out/r02ak_abn.txt
WV_LIB=var/sg2.so python profiles/timeline.py fp64 > gpurun_out/timeline_r02ak_sg2_fp64.txt 2>&1; tail -2 gpurun_out/timeline_r02ak_sg2_fp64.txt
