# k_row min-blocks experiment sweep (rebuilds the library on the box).
run() { for wl in cfg3 cfg4 cfg5; do python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $wl ms %.4f'%d['ms_per_step'], d['clocks']['sm_mhz'])"; done; }
for mb in 1 3 4 3 1; do
  RNT_NVCC_EXTRA="-DRNT_ROW_MINB=$mb" python -m paper_2410_05934_b200.build --force > /dev/null
  run minb$mb
done
