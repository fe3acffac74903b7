set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "external_product" 2>&1 | tail -3
for v in 1 0 -1; do RNT_EXTPROD=$v python bench.py --extprod --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('EXTPROD=$v', {k: (round(v['ms'],4), round(v['frac_alu'],3)) for k,v in d['results'].items()})"; done
python bench.py --extprod --steps 20 2>&1 | tail -1 > gpurun_out/bench_extprod.json
ncu --set full --clock-control none -k regex:"k_extprod" -s 2 -c 1 -o /tmp/prof_ext python -c "
import sys; sys.argv=['bench.py','--extprod','--steps','1','--warmup','1']; import runpy; runpy.run_path('bench.py', run_name='__main__')" > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_extprod_cta /tmp/prof_ext.ncu-rep
cat gpurun_out/ncu_extprod_cta.md
