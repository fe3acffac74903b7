for v in 0 1 2 3 4; do
  RNT_SMALL_VARIANT=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pb=d['parts'][1]
print('variant $v', 'partB_ms %.4f'%pb['ms'], 'frac %.3f'%pb['frac_alu'], 'partA_ms %.4f'%d['parts'][0]['ms'])
"
done
