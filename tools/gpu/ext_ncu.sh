ncu --set full --clock-control none -k regex:"k_extprod" -s 2 -c 1 -o /tmp/prof_ext python -c "
import sys; sys.argv=['bench.py','--extprod','--steps','1','--warmup','1']; import runpy; runpy.run_path('bench.py', run_name='__main__')" > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_extprod_cta /tmp/prof_ext.ncu-rep
cat gpurun_out/ncu_extprod_cta.md
