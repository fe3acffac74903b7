set -x
timeout 900 python -m pytest tests/test_bench_contract.py -q 2>&1 | tail -2
python bench.py --workload cfg1 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_cfg1.json
python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_cfg5_nocpu.json
