# Cluster path: parity (direct + env variants) and f3 latency.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster or variants" 2>&1 | tail -3
python bench.py --latency --steps 200 --warmup 10 2>&1 | tail -1
RNT_CLUSTER_C=8 python bench.py --latency --steps 200 --warmup 10 2>&1 | tail -1
RNT_CLUSTER_UNITS=0 python bench.py --latency --steps 200 --warmup 10 2>&1 | tail -1
