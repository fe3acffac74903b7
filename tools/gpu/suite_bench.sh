# Full GPU suite, then the default bench line and cfg3.
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py --no-cpu-baseline > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json
python bench.py --workload cfg3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 ms %.4f frac %.3f'%(d['ms_per_step'], d['roofline']['frac']))"
