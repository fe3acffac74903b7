# refresh of profiles/r01 after the LZ + k_clat changes (ncu reports summarised on the box:
# gpurun_out/ must stay below 64 MiB)
set -x
mkdir -p gpurun_out/p2 /tmp/p2
python bench.py 2>&1 | tail -1 > gpurun_out/p2/bench_cfg5.json
for w in cfg1 cfg2 cfg3 cfg4; do python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/p2/bench_$w.json; done
python bench.py --latency 2>&1 | tail -1 > gpurun_out/p2/bench_latency.json
python bench.py --keyswitch --steps 10 2>&1 | tail -1 > gpurun_out/p2/bench_keyswitch.json
python bench.py --extprod --steps 20 2>&1 | tail -1 > gpurun_out/p2/bench_extprod.json
python bench.py --modup --steps 20 2>&1 | tail -1 > gpurun_out/p2/bench_modup.json
python bench.py --automorph --steps 20 2>&1 | tail -1 > gpurun_out/p2/bench_automorph.json
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/p2/bench_reference.json
for w in cfg3 cfg5; do RNT_CLUSTER_UNITS=100 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CLUSTER_UNITS=100 $w', d['ms_per_step'], [(p['log2n'], round(p['ms'],4)) for p in d['parts']])"; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/p2/launches_cfg5.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_row|k_col" -s 4 -c 4 -o /tmp/p2/prof_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p2/ncu_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_clat|k_cluster" -c 5 -o /tmp/p2/prof_lat python tools/gpu/lat_kernels.py > gpurun_out/p2/ncu_lat.log 2>&1
python tools/ncu_summary.py gpurun_out/p2/ncu_full_cfg5 /tmp/p2/prof_cfg5.ncu-rep
python tools/ncu_summary.py gpurun_out/p2/ncu_full_lat /tmp/p2/prof_lat.ncu-rep
ncu -i /tmp/p2/prof_cfg5.ncu-rep --page source --csv -k regex:k_warp > /tmp/p2/src.csv 2>/dev/null; gzip -c /tmp/p2/src.csv > gpurun_out/p2/k_warp_source.csv.gz
ls -la gpurun_out/p2; du -sh gpurun_out
