# r02am: thinner heavy-piece / multi-row grids so the single-row tiles keep SM slots beside them
cd $GRAFT_REPO_ROOT
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/hp148.so var/hp296.so var/hp148m0.so var/hp296m2.so" bash profiles/abn.sh > gpurun_out/r02am_abn.txt 2>&1
cat gpurun_out/r02am_abn.txt
