# r02af: north_star target end to end on one B200 with the r02ac build (fp64, one global permutation)
cd $GRAFT_REPO_ROOT
timeout 1200 python profiles/northstar_e2e.py 10000000 0 fp64 > gpurun_out/northstar_e2e_r02af_fp64.json 2> gpurun_out/northstar_e2e_r02af_fp64.err
tail -c 1500 gpurun_out/northstar_e2e_r02af_fp64.json; tail -5 gpurun_out/northstar_e2e_r02af_fp64.err
