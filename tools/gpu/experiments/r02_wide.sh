# N = 2^16 path choice for small jobs: warp-engine rows (k_rows) with 8-column tiles, 2-warp teams
set -x
O=gpurun_out/r02k; mkdir -p $O
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1; }
summ() { python -c "
import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), [round(p['ms'],4) for p in d['parts']], d.get('digests_ok'))
    except Exception as e: print(f, 'ERR', e)
" "$@"; }
for v in "def:" "wide:-DRNT_WIDE_UNITS=3" "wideteam:-DRNT_WIDE_UNITS=3 -DRNT_ROWS_TEAM=2" "team:-DRNT_ROWS_TEAM=2"; do
  n=${v%%:*}; f=${v#*:}
  build "$f"
  for w in cfg3 cfg4 cfg5; do python bench.py --workload $w --steps 40 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_$n.json 2>&1; done
done
build ""
summ $O/bench_cfg*.json
