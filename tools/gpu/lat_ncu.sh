# Kernel-only durations of the single-polynomial forward NTT: cluster C=16 / C=8 / three-kernel path.
for cfg in "RNT_CLUSTER_C=16" "RNT_CLUSTER_C=8" "RNT_CLUSTER_UNITS=0"; do
  env $cfg ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/gpu/lat_kernels.py 2>/dev/null | python -c "
import csv, sys, collections
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
h = rows[0]; d = [dict(zip(h, r)) for r in rows[1:]]
out = collections.OrderedDict()
for x in d:
    name = x['Kernel Name'].split('(')[0].replace('void ', '')
    out.setdefault(name, []).append(float(x['Metric Value'].replace(',', '')))
print('$cfg', {k: round(min(v) / 1000, 2) for k, v in out.items()})
"
done
