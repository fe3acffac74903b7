# k_clat (latency cluster kernel): parity, latency A/B vs k_cluster
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_path or variants" 2>&1 | tail -3
for env in "RNT_CLAT=0" "RNT_CLAT=1" "RNT_CLAT_E=8" "RNT_CLAT_E=4" "RNT_CLAT_C=8" "RNT_CLAT_C=16"; do
  env $env python bench.py --latency 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', {k: round(v['us_graph'],2) for k,v in d['results'].items()})"
done
python bench.py --latency 2>&1 | tail -1 > gpurun_out/bench_latency.json
