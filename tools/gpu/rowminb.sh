set -x
run() { python bench.py --workload $1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2 $1', round(d['ms_per_step'],4), [(p['log2n'], round(p['ms'],4)) for p in d['parts']])"; }
for w in cfg3 cfg4 cfg5; do run $w default; done
for v in 1 2 3 4 5; do for w in cfg3 cfg5; do RNT_LARGE_VARIANT=$v run $w "LV=$v"; done; done
cp paper_2410_05934_b200/librnsntt.so /tmp/orig.so
RNT_NVCC_EXTRA=-DRNT_ROW_MINB=3 python -m paper_2410_05934_b200.build --force > /dev/null 2>&1
for w in cfg3 cfg4 cfg5; do run $w ROW_MINB3; done
cp /tmp/orig.so paper_2410_05934_b200/librnsntt.so
