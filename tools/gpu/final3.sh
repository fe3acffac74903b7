timeout 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
python __graft_entry__.py --smoke 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/final3_cfg5.json
python -c "import json; d=json.load(open('gpurun_out/final3_cfg5.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
