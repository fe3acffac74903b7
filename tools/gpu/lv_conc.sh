run() { python bench.py --no-cpu-baseline --no-e2e $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), [(p['log2n'], round(p['ms'],4)) for p in d['parts']])"; }
for i in 1 2; do
run default
for v in 1 4 5; do RNT_LARGE_VARIANT=$v run "LV=$v"; done
RNT_SPLIT=0 run "SPLIT=0"
RNT_SPLIT=3 run "SPLIT=3"
done
