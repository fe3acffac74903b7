# warp engine: group-loop unroll of the K = 2 passes
set -x
O=gpurun_out/r02j; mkdir -p $O
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1; }
summ() { python -c "
import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), [round(p['ms'],4) for p in d['parts']], d.get('digests_ok'))
    except Exception as e: print(f, 'ERR', e)
" "$@"; }
for v in 1 2; do
  build "-DRNT_K2_UNROLL=$v"
  for w in cfg5 cfg2 cfg4; do python bench.py --workload $w --steps 40 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_k2u$v.json 2>&1; done
  python bench.py --extprod --steps 20 > $O/bench_extprod_k2u$v.json 2>&1
done
build ""
summ $O/bench_cfg*.json
grep -h '"results"' $O/bench_extprod*.json | python -c "
import json,sys
for ln in sys.stdin: d=json.loads(ln); print({k:(round(v['ms'],4), round(v['frac_alu'],3)) for k,v in d['results'].items()})"
