# validation: team paths for every N=2^10 mode + bench lines with the new roofline fields
set -x
O=gpurun_out/r02w; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
for w in cfg5 cfg2; do python bench.py --workload $w --steps 30 --no-cpu-baseline > $O/bench_$w.json 2>&1; done
python bench.py --extprod --steps 20 > $O/bench_extprod.json 2>&1
python -c "
import json
for f in ['$O/bench_cfg5.json','$O/bench_cfg2.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']; print(f, d['value']/1e6, d['ms_per_step'], r['frac'], r['frac_incl_pointwise'], d['digests_ok'])
d=json.loads(open('$O/bench_extprod.json').read().strip().splitlines()[-1]); print({k:(round(v['ms'],4), round(v['frac_alu'],3), round(v['frac_alu_incl_mac'],3)) for k,v in d['results'].items()})
"
