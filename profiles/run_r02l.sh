# r02l: quoted-csv ingest + walks + formats parity; cfg5 walk kernel ncu with the walk adjacency;
# owner L2-prefetch A/B (fp64)
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_ingest.py tests/test_gpu_walks.py tests/test_gpu_formats.py tests/test_gpu_synth.py -q > gpurun_out/r02l_tests.log 2>&1; tail -3 gpurun_out/r02l_tests.log
OUT=gpurun_out/prof_random_walk_kernel_cfg5_r02l
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:random_walk_kernel -s 1 -c 1 -o $OUT -f python profiles/cfg5_walk_prof.py > $OUT.log 2>&1
ncu -i $OUT.ncu-rep --page details --csv > $OUT.details.csv 2>/dev/null
ncu -i $OUT.ncu-rep --page raw --csv > $OUT.raw.csv 2>/dev/null
gzip -f $OUT.raw.csv; rm -f $OUT.ncu-rep
LIBS="var/cur.so var/fpf1.so var/fpf2.so" bash profiles/abn.sh > gpurun_out/r02l_abn.txt 2>&1
