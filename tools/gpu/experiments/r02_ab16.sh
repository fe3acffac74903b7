# A/B for the N = 2^16 part: two-pass chain (default) vs the single-launch cluster kernel
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r02d_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r02d_pytest_gpu.txt
set -x
O=gpurun_out/r02d; mkdir -p $O /tmp/r02d
for w in cfg3 cfg4; do
  python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}.json 2>&1
  RNT_CLUSTER_UNITS=1000 python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_cluster.json 2>&1
done
RNT_CLUSTER_UNITS=1000 python bench.py --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_cfg5_cluster.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_col|k_row|k_cluster" -c 4 -o /tmp/r02d/prof16 python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/ncu16.log 2>&1
RNT_CLUSTER_UNITS=1000 ncu --set full --clock-control none --import-source on -k regex:"k_cluster" -c 1 -o /tmp/r02d/profcl python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/ncucl.log 2>&1
python tools/ncu_summary.py $O/ncu_16 /tmp/r02d/prof16.ncu-rep /tmp/r02d/profcl.ncu-rep > /dev/null 2>&1
ls -la /tmp/r02d
for f in $O/bench_*.json; do echo $f; python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], [p['ms'] for p in d['parts']], d['digests_ok'])"; done
ncu --set full --clock-control none --import-source on -k regex:"k_hrf" -c 1 -o /tmp/r02d/profhrf python bench.py --hrf --steps 1 --warmup 1 > $O/ncuhrf.log 2>&1
python tools/ncu_summary.py $O/ncu_hrf /tmp/r02d/profhrf.ncu-rep > /dev/null 2>&1
ncu -i /tmp/r02d/profhrf.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keys=[k for k in h if k.startswith('dram__') or 'lts__t_sectors_srcunit_tex_op_read' in k or 'long_scoreboard' in k or 'sm__warps_active' in k]
for row in r[2:]:
    d=dict(zip(h,row)); print(d['Kernel Name'][:40]); [print(' ',k,d[k]) for k in keys]
" > $O/hrf_dram.txt

for u in 8 2; do
RNT_NVCC_EXTRA="-DRNT_HRF_UNROLL=$u" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
python bench.py --hrf --steps 10 > $O/bench_hrf_u$u.json 2>&1
done
RNT_NVCC_EXTRA="-DRNT_HRF_CTAS_PER_SM=4" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
python bench.py --hrf --steps 10 > $O/bench_hrf_c4.json 2>&1
python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
