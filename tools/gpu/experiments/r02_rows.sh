# cfg4 wide path: k_rows with 2-warp teams and 32 warps/SM; extprod / cfg5 / cfg2 with the new default
set -x
O=gpurun_out/r02n; mkdir -p $O
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > $O/build_$2.txt 2>&1; }
summ() { python -c "
import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), [round(p['ms'],4) for p in d['parts']], d.get('digests_ok'))
    except Exception as e: print(f, 'ERR', e)
" "$@"; }
for v in "def:" "t2m16:-DRNT_ROWS_TEAM=2 -DRNT_ROWS_MINB=16" "t2m12:-DRNT_ROWS_TEAM=2" "t1m16:-DRNT_ROWS_MINB=16"; do
  n=${v%%:*}; f=${v#*:}
  build "$f" $n
  python bench.py --workload cfg4 --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_cfg4_$n.json 2>&1
done
build "" def2
for w in cfg5 cfg2; do python bench.py --workload $w --steps 40 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_new.json 2>&1; done
summ $O/bench_cfg*.json
