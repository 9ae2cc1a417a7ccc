# r02z: fp64 update-phase A/B on the r02y defaults: heavy-piece loads / grids (p0-p2), multi rows per SM (p3),
# grouped contribution loads in the multi-contribution owner (g2, g4, g4m3)
cd $GRAFT_REPO_ROOT
LIBS="paper_2508_01073_b200/libwalkvec_b200.so var/p0.so var/p1.so var/p2.so var/p3.so var/g2.so var/g4.so var/g4m3.so" bash profiles/abn.sh > gpurun_out/r02z_abn.txt 2>&1
cat gpurun_out/r02z_abn.txt
WV_LIB=var/g4m3.so python profiles/timeline.py fp64 > gpurun_out/timeline_r02z_g4m3_fp64.txt 2>&1; tail -2 gpurun_out/timeline_r02z_g4m3_fp64.txt
WV_LIB=var/g4m3.so timeout 600 bash profiles/ncu_one.sh sgns_owner_flat_kernel r02z_g4m3
python profiles/ncu_brief.py gpurun_out/prof_sgns_owner_flat_kernel_r02z_g4m3.details.csv
