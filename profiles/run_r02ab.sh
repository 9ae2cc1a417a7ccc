# r02ab: concurrent singles tile size (items per thread per CTA) 8 .. 32 vs the serial schedule
cd $GRAFT_REPO_ROOT
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/t12.so var/t16.so var/t24.so var/t32.so" bash profiles/abn.sh > gpurun_out/r02ab_abn.txt 2>&1
cat gpurun_out/r02ab_abn.txt
