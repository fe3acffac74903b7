# round 2, A/B batch 2: tests, 2^16 two-pass vs cluster, warp teams for the cfg2 tail, HRF unroll/occupancy
set -x
O=gpurun_out/r02e; mkdir -p $O /tmp/r02e
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1; }
summ() { python -c "
import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), [round(p['ms'],4) for p in d['parts']], d.get('digests_ok'))
    except Exception as e: print(f, 'ERR', e)
" "$@"; }
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
for w in cfg2 cfg3 cfg4 cfg5; do python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}.json 2>&1; done
for w in cfg3 cfg4 cfg5; do RNT_CLUSTER_UNITS=1000 python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_cluster.json 2>&1; done
ncu --set full --clock-control none -k regex:"k_col|k_row|k_cluster" -c 4 -o /tmp/r02e/prof16 python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
RNT_CLUSTER_UNITS=1000 ncu --set full --clock-control none -k regex:"k_cluster" -c 1 -o /tmp/r02e/profcl python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_hrf" -c 1 -o /tmp/r02e/profhrf python bench.py --hrf --steps 1 --warmup 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_16 /tmp/r02e/prof16.ncu-rep /tmp/r02e/profcl.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_hrf /tmp/r02e/profhrf.ncu-rep > /dev/null 2>&1
ncu -i /tmp/r02e/profhrf.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keys=[k for k in h if k.startswith('dram__') or 'long_scoreboard' in k or 'sm__warps_active' in k or 'l1tex__t_bytes' in k]
for row in r[2:]:
    d=dict(zip(h,row)); print(d['Kernel Name'][:40]); [print(' ',k,d[k]) for k in keys]
" > $O/hrf_metrics.txt
python bench.py --hrf --steps 10 > $O/bench_hrf.json 2>&1
for u in 8 2; do build "-DRNT_HRF_UNROLL=$u"; python bench.py --hrf --steps 10 > $O/bench_hrf_u$u.json 2>&1; done
build "-DRNT_HRF_CTAS_PER_SM=4"; python bench.py --hrf --steps 10 > $O/bench_hrf_c4.json 2>&1
build "-DRNT_HRF_CTAS_PER_SM=16"; python bench.py --hrf --steps 10 > $O/bench_hrf_c16.json 2>&1
build "-DRNT_TEAM2_WAVES=100"; for w in cfg2 cfg5; do python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_team2.json 2>&1; done
build "-DRNT_TEAM4_WAVES=100"; for w in cfg2 cfg5; do python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_team4.json 2>&1; done
build ""
summ $O/bench_cfg*.json
grep -h '"results"' $O/bench_hrf*.json | python -c "
import json,sys
for ln in sys.stdin: d=json.loads(ln); print({k:(round(v['ms'],4), round(v['frac_hbm'],3)) for k,v in d['results'].items()})"
