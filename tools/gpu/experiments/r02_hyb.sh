# hybrid integer / FP64 Shoup butterfly microbenchmark + pipe counters
O=gpurun_out/hyb; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
for c in 2 3 4; do ./tools/microbench/hyb $c; done > $O/hyb.jsonl 2>&1
cat $O/hyb.jsonl
ncu --clock-control none --metrics regex:sm__inst_executed_pipe_.*,regex:sm__pipe_.*_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg --csv ./tools/microbench/hyb 4 > $O/hyb_ncu.csv 2> $O/hyb_ncu.err
python3 - <<'PY' > $O/hyb_pipes.txt
import csv
rows = list(csv.reader(open('gpurun_out/hyb/hyb_ncu.csv')))
hdr = None
out = {}
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if not hdr or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    k = d['ID'] + ' ' + d['Kernel Name'][:40]
    try: v = float(d['Metric Value'].replace(',', ''))
    except: continue
    if v == 0: continue
    out.setdefault(k, []).append((d['Metric Name'], v))
for k, ms in out.items():
    print(k)
    for m, v in ms: print('   ', m, v)
PY
head -150 $O/hyb_pipes.txt
