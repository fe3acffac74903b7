# round-2 baseline on the GPU box: metric names, bench lines, launch list, ncu full capture
set -x
O=gpurun_out/r02a; mkdir -p $O /tmp/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
ncu --query-metrics --chip gb100 2>/dev/null | grep -iE "pipe_(fmaheavy|alu|fma)|bank_conflicts|wavefronts_mem_shared" > $O/metric_names.txt
python bench.py --steps 50 --warmup 5 2>&1 | tail -1 > $O/bench_cfg5.json
for w in cfg2 cfg3 cfg4; do python bench.py --workload $w --no-cpu-baseline --steps 50 2>&1 | tail -1 > $O/bench_$w.json; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_row|k_col" -s 4 -c 4 -o /tmp/r02a/prof_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_cfg5.log 2>&1
python tools/ncu_summary.py $O/ncu_full_cfg5 /tmp/r02a/prof_cfg5.ncu-rep > /dev/null
cp /tmp/r02a/prof_cfg5.ncu-rep $O/ 
ls -la $O
