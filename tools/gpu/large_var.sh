run() { for wl in cfg3 cfg4 cfg5; do env $2 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $wl ms %.4f'%d['ms_per_step'])"; done; }
run default ""
for v in 1 2 4 5 6; do run v$v "RNT_LARGE_VARIANT=$v"; done
run split3 "RNT_SPLIT=3"
run split4 "RNT_SPLIT=4"
