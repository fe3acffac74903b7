# swizzled warp buffers + HRF + pruned variants: tests, bench, ncu of k_warp
set -x
O=gpurun_out/r02c; mkdir -p $O /tmp/r02c
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -5 $O/pytest_gpu.txt
python __graft_entry__.py --smoke > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
python bench.py --workload cfg2 --steps 50 --no-cpu-baseline > $O/bench_cfg2.json 2>&1
python bench.py --hrf --steps 10 > $O/bench_hrf.json 2>&1
python bench.py --extprod --steps 20 > $O/bench_extprod.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_hrf" -c 2 -o /tmp/r02c/prof python bench.py --workload cfg2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/ncu_kwarp /tmp/r02c/prof.ncu-rep > /dev/null 2>&1
cp /tmp/r02c/prof.ncu-rep $O/
tail -3 $O/*.json
# A/B: 28 warps/SM (14 CTAs, <= 72 registers) -- one wave for cfg2's 4096 polynomials
RNT_NVCC_EXTRA="-DRNT_WARP_MINB=14" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > $O/build14.txt 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/bench_cfg5_minb14.json 2>&1
python bench.py --workload cfg2 --steps 50 --no-cpu-baseline --no-e2e --no-graph > $O/bench_cfg2_minb14.json 2>&1
RNT_NVCC_EXTRA="-DRNT_WARP_MINB=13" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > $O/build13.txt 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/bench_cfg5_minb13.json 2>&1
python bench.py --workload cfg2 --steps 50 --no-cpu-baseline --no-e2e --no-graph > $O/bench_cfg2_minb13.json 2>&1
python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
RNT_BENCH_SHARE_GPU=1 timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_share2.json 2> $O/bench_share2.err
tail -c 400 $O/bench_share2.json
