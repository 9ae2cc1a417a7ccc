# r02x: fp64 A/B: a (shared exp) vs e (+ reciprocal bias corrections), f (heavy then multi rows serially),
# g (10x2 gather ring + low-priority side stream), h (multi-contribution rows at 2 CTAs/SM), c (10x2 ring)
cd $GRAFT_REPO_ROOT
LIBS="var/a.so var/e.so var/f.so var/g.so var/h.so var/c.so" bash profiles/abn.sh > gpurun_out/r02x_abn.txt 2>&1
cat gpurun_out/r02x_abn.txt
WV_LIB=var/e.so timeout 600 bash profiles/ncu_one.sh sgns_owner_single_kernel r02x_e
python profiles/ncu_brief.py gpurun_out/prof_sgns_owner_single_kernel_r02x_e.details.csv
