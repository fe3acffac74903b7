# session 3 start: verify HEAD on the GPU (tests, smoke, bench lines)
O=gpurun_out/r02v; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
python __graft_entry__.py --smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py --steps 50 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for w in cfg2 cfg3 cfg4; do python bench.py --workload $w --steps 50 --no-cpu-baseline > $O/bench_$w.json 2>&1; done
python bench.py --keyswitch --steps 10 > $O/bench_keyswitch.json 2>&1
python bench.py --extprod --steps 20 > $O/bench_extprod.json 2>&1
ls -la $O
