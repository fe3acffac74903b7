"""Print the per-kernel launch list of the last key switch in an ncu CSV
(tools/gpu/ks.sh): duration and DRAM bytes per launch."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    agg.setdefault((d["ID"], d["Kernel Name"][:60]), {})[d["Metric Name"]] = d["Metric Value"]
items = list(agg.items())
per = int(sys.argv[2]) if len(sys.argv) > 2 else len(items) // 3
tot = 0.0
for (i, name), m in items[-per:]:
    f = lambda k: float(m[k].replace(",", ""))
    t = f("gpu__time_duration.sum") / 1000
    tot += t
    print(f"{name:60s} {t:9.1f} us  R {f('dram__bytes_read.sum') / 1e6:8.1f} MB  W {f('dram__bytes_write.sum') / 1e6:8.1f} MB")
print(f"total {tot:.1f} us")
