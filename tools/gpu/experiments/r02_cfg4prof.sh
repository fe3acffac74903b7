# cfg4 kernel shares and pipe utilisation (wide path: 8-column tiles + k_rows)
set -x
O=gpurun_out/r02x; mkdir -p $O /tmp/r02x
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_cfg4.csv python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_col|k_rows" -s 3 -c 3 -o /tmp/r02x/cfg4 python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_cfg4 /tmp/r02x/cfg4.ncu-rep > /dev/null 2>&1
cat $O/ncu_cfg4.md
