timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -4
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms/step',d['ms_per_step'],'roof',d['roofline']['frac'], 'clk', d['clocks'])
for p in d['parts']: print(p)
"
