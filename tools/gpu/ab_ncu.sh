# A/B kernel durations (ncu launch list) for cfg4: current tree vs tmp_ab/old.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_new.csv python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
(cd tmp_ab/old && python -m paper_2410_05934_b200.build --force > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $GRAFT_REPO_ROOT/gpurun_out/ab_old.csv python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1)
for f in new old; do python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/ab_$f.csv")) if len(r)>10]
h=rows[0]; d=[dict(zip(h,r)) for r in rows[1:]]
import collections
agg=collections.defaultdict(list)
for x in d: agg[x['Kernel Name'][:40]].append(float(x['Metric Value'].replace(',','')))
for k,v in agg.items(): print("$f", k, len(v), round(sum(v[-3:])/3/1000,1), 'us (last 3 avg)')
PY
done
