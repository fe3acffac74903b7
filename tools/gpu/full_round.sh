# parity + bench + ncu evidence for profiles/
set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3
python __graft_entry__.py --smoke 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/bench_cfg5.json
cat gpurun_out/bench_cfg5.json
for w in cfg2 cfg3 cfg4; do python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$w.json; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_row|k_col" -s 4 -c 4 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
