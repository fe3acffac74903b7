# dataflow 2^16 polymul (k_flow) vs the three-kernel chain
set -x
O=gpurun_out/r02h; mkdir -p $O /tmp/r02g
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1; }
summ() { python -c "
import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), [round(p['ms'],4) for p in d['parts']], d.get('digests_ok'))
    except Exception as e: print(f, 'ERR', e)
" "$@"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "16 or cfg or bench or polymul or variants or automorph" > $O/pytest_parity.txt 2>&1; tail -3 $O/pytest_parity.txt
for w in cfg3 cfg4 cfg5; do python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_flow.json 2>&1; done
ncu --set full --clock-control none -k regex:"k_flow" -c 1 -o /tmp/r02g/flow python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_flow /tmp/r02g/flow.ncu-rep > /dev/null 2>&1
build "-DRNT_FLOW=0"
for w in cfg3 cfg4 cfg5; do python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_chain.json 2>&1; done
build ""
python bench.py --automorph --steps 20 > $O/bench_automorph.json 2>&1; tail -c 400 $O/bench_automorph.json
summ $O/bench_*.json
cat $O/ncu_flow.md
