# Round-end evidence refresh: bench lines for every mode, launch list, ncu captures.
mkdir -p gpurun_out/r01b
O=gpurun_out/r01b
python bench.py > $O/bench_cfg5.json 2>$O/err.txt
for w in cfg1 cfg2 cfg3 cfg4; do python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2>>$O/err.txt; done
python bench.py --latency > $O/bench_latency.json 2>>$O/err.txt
python bench.py --automorph --steps 20 > $O/bench_automorph.json 2>>$O/err.txt
python bench.py --extprod --steps 20 > $O/bench_extprod.json 2>>$O/err.txt
python bench.py --modup --steps 20 > $O/bench_modup.json 2>>$O/err.txt
python bench.py --keyswitch --steps 10 > $O/bench_keyswitch.json 2>>$O/err.txt
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>>$O/err.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
XM=sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active
ncu --set full --metrics $XM --clock-control none --import-source on -k regex:"k_warp|k_row|k_col" -s 21 -c 7 -o /tmp/prof_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_cfg5.log 2>&1
ncu --set full --metrics $XM --clock-control none -k regex:"k_cluster" -c 3 -o /tmp/prof_cluster python tools/gpu/lat_kernels.py > /dev/null 2>&1
ncu --set full --metrics $XM --clock-control none -k regex:"k_row_mac|k_col_fwd" -s 2 -c 2 -o /tmp/prof_ks python tools/gpu/ks1.py > /dev/null 2>&1 || true
python tools/ncu_summary.py $O/ncu_full_cfg5 /tmp/prof_cfg5.ncu-rep > /dev/null
python tools/ncu_summary.py $O/ncu_full_cluster /tmp/prof_cluster.ncu-rep > /dev/null
python tools/ncu_summary.py $O/ncu_full_keyswitch /tmp/prof_ks.ncu-rep > /dev/null
ls -la $O
