set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_path or variants" 2>&1 | tail -3
python bench.py --latency 2>&1 | tail -1 | tee gpurun_out/bench_latency.json
RNT_CLAT=0 python bench.py --latency 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('k_cluster', {k: round(v['us_graph'],2) for k,v in d['results'].items()})"
for w in cfg3 cfg5; do python bench.py --workload $w --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default $w', d['ms_per_step'], [(p['log2n'], round(p['ms'],4)) for p in d['parts']])"; done
cp paper_2410_05934_b200/librnsntt.so /tmp/orig.so
RNT_NVCC_EXTRA=-DRNT_COL_MINB=4 python -m paper_2410_05934_b200.build --force > /dev/null 2>&1
for w in cfg3 cfg5 cfg4; do python bench.py --workload $w --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('COL_MINB=4 $w', d['ms_per_step'], [(p['log2n'], round(p['ms'],4)) for p in d['parts']])"; done
cp /tmp/orig.so paper_2410_05934_b200/librnsntt.so
python bench.py --workload cfg4 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default cfg4', d['ms_per_step'])"
