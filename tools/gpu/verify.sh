# quick state check: GPU parity, smoke, default bench line, cfg1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3
python __graft_entry__.py --smoke 2>&1 | tail -1
python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_cfg5.json
python bench.py --workload cfg1 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_cfg1.json
python bench.py --workload cfg3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_cfg3.json
