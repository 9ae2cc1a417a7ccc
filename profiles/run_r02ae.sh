# r02ae: occupancy of the single-contribution row tiles: 4 CTAs/SM (64 registers) vs 5 / 6
cd $GRAFT_REPO_ROOT
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/m5.so var/m6.so var/m5t16.so" bash profiles/abn.sh > gpurun_out/r02ae_abn.txt 2>&1
cat gpurun_out/r02ae_abn.txt
