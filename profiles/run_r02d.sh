# r02d: A/B of gather L2 prefetch / owner grid / two items per owner thread / heavy-piece grid (fp64 cfg2),
# and the multi-rank device tests
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_dist_gpu.py tests/test_shard_gpu.py -q > gpurun_out/r02d_dist_tests.log 2>&1
LIBS="var/gpf0.so var/gpf2.so var/gpf4.so var/gpf8.so var/own5.so var/flatu2.so var/pg296.so" bash profiles/abn.sh > gpurun_out/r02d_abn.txt 2>&1
