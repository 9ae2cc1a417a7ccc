# r02h: heavy pieces with all group loads in flight (hp), with the 64-register light owner at 3 CTAs/SM
# (m4p3) and with a 296-CTA piece grid; fp64 and fp32 cfg2
cd $GRAFT_REPO_ROOT
LIBS="var/base.so var/m4p3.so var/hp.so var/hpm4p3.so var/hppg.so" bash profiles/abn.sh > gpurun_out/r02h_abn64.txt 2>&1
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 --precision fp32" LIBS="var/base.so var/m4p3.so var/hp.so var/hpm4p3.so" bash profiles/abn.sh > gpurun_out/r02h_abn32.txt 2>&1
python -m pytest tests/test_gpu_formats.py -q > gpurun_out/r02h_formats.log 2>&1
