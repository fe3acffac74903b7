for v in 11 13; do RNT_SMALL_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "all_sizes or cfg2 or edge or in_place or roundtrip" 2>&1 | tail -1; done
for v in 8 11 12 13 14; do
  RNT_SMALL_VARIANT=$v python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pb=d['parts'][1]
print('variant $v', 'partB_ms %.4f'%pb['ms'], 'frac %.3f'%pb['frac_alu'])
"
done
