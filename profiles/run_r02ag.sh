# r02ag: fp64 streaming (evict-first) stores of the updated rows: m, v (s1), p + m + v (s2), p (s3)
cd $GRAFT_REPO_ROOT
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/s1.so var/s2.so var/s3.so" bash profiles/abn.sh > gpurun_out/r02ag_abn.txt 2>&1
cat gpurun_out/r02ag_abn.txt
