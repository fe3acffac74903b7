# bench.py multi-rank plumbing on a 1-GPU box (ranks share the GPU over gloo) + the default line
set -x
O=gpurun_out/r02b; mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
RNT_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_share2.json 2> $O/bench_share2.err
RNT_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --scaling weak > $O/bench_share2_weak.json 2> $O/bench_share2_weak.err
python bench.py --workload cfg1 --steps 20 --no-cpu-baseline > $O/bench_cfg1.json 2>&1
timeout 900 python -m pytest tests/test_bench_contract.py -q -x > $O/pytest_contract.txt 2>&1
tail -3 $O/*.err $O/pytest_contract.txt
