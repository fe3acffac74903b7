set -x
python bench.py --steps 10 --warmup 3 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_team -s 2 -c 1 -o gpurun_out/prof_team python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_team.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_row -s 2 -c 1 -o gpurun_out/prof_row python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_row.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_col -s 4 -c 2 -o gpurun_out/prof_col python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_col.log 2>&1
ls -la gpurun_out
