# Cluster path for batched large-N jobs vs the split three-kernel path.
run() { for wl in cfg3 cfg4 cfg5; do env $2 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $wl ms %.4f'%d['ms_per_step'])"; done; }
run default ""
run cl16 "RNT_CLUSTER_UNITS=100000 RNT_CLUSTER_C=16"
run cl16_nosplit "RNT_CLUSTER_UNITS=100000 RNT_CLUSTER_C=16 RNT_SPLIT=0"
run cl8 "RNT_CLUSTER_UNITS=100000 RNT_CLUSTER_C=8"
