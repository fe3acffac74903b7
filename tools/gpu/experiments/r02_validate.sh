# validation of the current tree: GPU tests, smoke, default bench line, 2-rank shared-GPU run
set -x
O=gpurun_out/r02v; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
python __graft_entry__.py --smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.json
RNT_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_share2.json 2> $O/bench_share2.err; tail -c 300 $O/bench_share2.json
