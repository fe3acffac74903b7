# round-2 evidence: every bench line, launch list, ncu full of the dominant kernels, sanitizer, tests
set -x
O=gpurun_out/r02s4; mkdir -p $O /tmp/r02z
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
lscpu | head -20 > $O/lscpu.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
python __graft_entry__.py --smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py --steps 50 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_cfg5_b.json 2>&1
for w in cfg1 cfg2 cfg3 cfg4; do python bench.py --workload $w --steps 50 --no-cpu-baseline > $O/bench_$w.json 2>&1; done
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1
python bench.py --latency > $O/bench_latency.json 2>&1
python bench.py --automorph --steps 20 > $O/bench_automorph.json 2>&1
python bench.py --extprod --steps 20 > $O/bench_extprod.json 2>&1
python bench.py --hrf --steps 20 > $O/bench_hrf.json 2>&1
python bench.py --modup --steps 20 > $O/bench_modup.json 2>&1
python bench.py --keyswitch --steps 10 > $O/bench_keyswitch.json 2>&1
RNT_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_share2_strong.json 2> $O/bench_share2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_row|k_col" -s 4 -c 4 -o /tmp/r02z/cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_warp" -c 1 -o /tmp/r02z/cfg2 python bench.py --workload cfg2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_hrf|k_automorph|k_extprod" -c 3 --import-source on -o /tmp/r02z/next python -c "
import sys, runpy
for m in (['--hrf'], ['--automorph'], ['--extprod']):
    sys.argv = ['bench.py', *m, '--steps', '1', '--warmup', '1']; runpy.run_path('bench.py', run_name='__main__')" > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_full_cfg5 /tmp/r02z/cfg5.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_full_cfg2 /tmp/r02z/cfg2.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_full_next /tmp/r02z/next.ncu-rep > /dev/null 2>&1
ncu -i /tmp/r02z/cfg5.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, json, sys
r = list(csv.reader(sys.stdin)); h = r[0]; out = {}
for row in r[2:]:
    d = dict(zip(h, row)); nm = d['Kernel Name'][:60]
    out.setdefault(nm, {'dram_bytes_read': d.get('dram__bytes_read.sum'), 'dram_bytes_write': d.get('dram__bytes_write.sum'), 'unit_read': r[1][h.index('dram__bytes_read.sum')]})
json.dump(out, open('$O/ncu_traffic_cfg5.json', 'w'), indent=1)"
# compute-sanitizer is closed on this GPU pool (runs under it have left GPUs needing a reset):
# profiles/r02/final/sanitizer.txt is the earlier round-2 run.
ls -la $O
