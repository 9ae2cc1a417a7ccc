# r02ao: fp64 heavy-row piece size (16 / 32 / 64) and the light/heavy threshold (8 / 16 / 32 contributions)
cd $GRAFT_REPO_ROOT
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/pc64.so var/pc16.so var/lm32.so var/lm8.so" bash profiles/abn.sh > gpurun_out/r02ao_abn.txt 2>&1
cat gpurun_out/r02ao_abn.txt
