set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -2
python __graft_entry__.py --smoke 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/bench_cfg5.json
for w in cfg1 cfg2 cfg3 cfg4; do python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$w.json; done
python bench.py --latency 2>&1 | tail -1 > gpurun_out/bench_latency.json
python bench.py --automorph --steps 20 2>&1 | tail -1 > gpurun_out/bench_automorph.json
python bench.py --extprod --steps 20 2>&1 | tail -1 > gpurun_out/bench_extprod.json
python bench.py --modup --steps 20 2>&1 | tail -1 > gpurun_out/bench_modup.json
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_row|k_col" -s 4 -c 4 -o gpurun_out/prof_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_final.log 2>&1
ncu --set full --clock-control none -k regex:"k_extprod|k_bconv|k_automorph" -c 3 -o gpurun_out/prof_next python -c "
import sys; sys.argv=['bench.py','--extprod','--steps','1','--warmup','1']; import runpy; runpy.run_path('bench.py', run_name='__main__')" > /dev/null 2>&1
ls -la gpurun_out | tail -20
