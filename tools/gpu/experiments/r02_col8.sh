# cfg3 / cfg5: 8-column pass-1 tiles (twice the CTAs) with the 16-thread-per-row k_row
set -x
O=gpurun_out/r02q; mkdir -p $O
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > $O/build_$2.txt 2>&1; }
for v in "def:" "col8:-DRNT_COL8_UNITS=3"; do
  n=${v%%:*}; f=${v#*:}
  build "$f" $n
  for w in cfg3 cfg5; do python bench.py --workload $w --steps 40 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_$n.json 2>&1; done
done
build "" def2
python -c "
import json,glob
for f in sorted(glob.glob('$O/bench_cfg*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), [round(p['ms'],4) for p in d['parts']], d.get('digests_ok'))
"
