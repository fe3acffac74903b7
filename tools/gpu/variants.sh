timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for v in 1 2 3; do RNT_LARGE_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "all_sizes or cfg3 or edge or in_place" 2>&1 | tail -1; done
for v in 0 1 2 3; do
  RNT_LARGE_VARIANT=$v python bench.py --workload cfg3 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg3 largevar $v', 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
  RNT_LARGE_VARIANT=$v python bench.py --workload cfg4 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg4 largevar $v', 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
done
python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg5 default', 'ms %.4f'%d['ms_per_step'], 'value %.4e'%d['value'], [round(p['ms'],4) for p in d['parts']])"
