for v in 4 5; do RNT_LARGE_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "all_sizes or cfg3 or cfg4 or edge or in_place or roundtrip or chunked" 2>&1 | tail -1; done
for v in 0 4 5; do
  RNT_LARGE_VARIANT=$v python bench.py --workload cfg3 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg3 largevar $v', 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
  RNT_LARGE_VARIANT=$v python bench.py --workload cfg4 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg4 largevar $v', 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
done
