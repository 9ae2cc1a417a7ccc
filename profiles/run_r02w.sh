# r02w: shared exp in the fp64 loss/sigmoid (a vs nosexp), side stream after the gather (b, d), 10x2 gather ring (c, d)
cd $GRAFT_REPO_ROOT
LIBS="var/nosexp.so var/a.so var/b.so var/c.so var/d.so" bash profiles/abn.sh > gpurun_out/r02w_abn.txt 2>&1
cat gpurun_out/r02w_abn.txt
WV_LIB=var/b.so python profiles/timeline.py fp64 > gpurun_out/timeline_r02w_b_fp64.txt 2>&1; tail -2 gpurun_out/timeline_r02w_b_fp64.txt
WV_LIB=var/d.so python profiles/timeline.py fp64 > gpurun_out/timeline_r02w_d_fp64.txt 2>&1; tail -2 gpurun_out/timeline_r02w_d_fp64.txt
WV_LIB=var/c.so timeout 600 bash profiles/ncu_one.sh sgns_gather_bulk_kernel r02w_c
WV_LIB=var/a.so timeout 600 bash profiles/ncu_one.sh sgns_gather_bulk_kernel r02w_a
python profiles/ncu_brief.py gpurun_out/prof_sgns_gather_bulk_kernel_r02w_*.details.csv
