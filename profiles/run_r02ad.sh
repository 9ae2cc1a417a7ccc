# r02ad: fp64 L2 policy of the gather's copies: evict-last on all lines (default) vs none / half / quarter
cd $GRAFT_REPO_ROOT
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/k0.so var/k50.so var/k25.so" bash profiles/abn.sh > gpurun_out/r02ad_abn.txt 2>&1
cat gpurun_out/r02ad_abn.txt
