# r02aj: is the gather slower in the pipeline because of the L2 state or the concurrent side stream?
# ncu serialises kernels; --cache-control none keeps the L2 as the previous kernels left it
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for CC in none all; do
  timeout 900 ncu --metrics $M --clock-control none --cache-control $CC -k regex:"sgns_gather_bulk|sgns_owner_single" -s 600 -c 60 --csv --log-file gpurun_out/r02aj_cc_$CC.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --configs none --fp32-steps 0 > gpurun_out/r02aj_$CC.log 2>&1
done
python - <<'PY'
import csv, collections
for cc in ("none", "all"):
    rows = [r for r in csv.reader(open(f"gpurun_out/r02aj_cc_{cc}.csv")) if len(r) > 10]
    h = rows[0]; iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    acc = collections.defaultdict(list)
    for r in rows[1:]:
        acc[(r[iK][:30], r[iM])].append(float(r[iV].replace(",", "")))
    for k, v in sorted(acc.items()):
        print(cc, k, round(sum(v) / len(v), 2), len(v))
PY
