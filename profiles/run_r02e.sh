# r02e: pipelined-batch timelines (light owner vs heavy pieces), A/B of the fused heavy pieces and a
# 256-thread heavy-piece CTA (fp64 cfg2), then compute-sanitizer over the small workload
cd $GRAFT_REPO_ROOT
python profiles/timeline.py fp64 > gpurun_out/timeline_r02e_fp64.txt 2>&1
python profiles/timeline.py fp32 > gpurun_out/timeline_r02e_fp32.txt 2>&1
LIBS="var/base.so var/fused.so var/pt256.so" bash profiles/abn.sh > gpurun_out/r02e_abn.txt 2>&1
bash profiles/sanitize.sh > gpurun_out/r02e_sanitize.txt 2>&1
