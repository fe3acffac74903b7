set -x
mkdir -p gpurun_out/p4 /tmp/p4
python bench.py 2>&1 | tail -1 > gpurun_out/p4/bench_cfg5.json
for w in cfg1 cfg2 cfg3 cfg4; do python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/p4/bench_$w.json; done
python bench.py --latency 2>&1 | tail -1 > gpurun_out/p4/bench_latency.json
python bench.py --keyswitch --steps 10 2>&1 | tail -1 > gpurun_out/p4/bench_keyswitch.json
python bench.py --extprod --steps 20 2>&1 | tail -1 > gpurun_out/p4/bench_extprod.json
python bench.py --modup --steps 20 2>&1 | tail -1 > gpurun_out/p4/bench_modup.json
python bench.py --automorph --steps 20 2>&1 | tail -1 > gpurun_out/p4/bench_automorph.json
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/p4/bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/p4/launches_cfg5.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_row|k_col" -s 4 -c 4 -o /tmp/p4/prof_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p4/ncu_cfg5.log 2>&1
python tools/ncu_summary.py gpurun_out/p4/ncu_full_cfg5 /tmp/p4/prof_cfg5.ncu-rep
ncu -i /tmp/p4/prof_cfg5.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keys=[k for k in h if 'fmaheavy' in k or 'pipe_alu_cycles' in k or 'pipe_fma_cycles' in k]
for row in r[2:]:
    d=dict(zip(h,row)); print(d['Kernel Name'][:40], {k:d[k] for k in keys})
" > gpurun_out/p4/pipes.txt
ls -la gpurun_out/p4
