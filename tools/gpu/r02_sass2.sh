O=gpurun_out/sass2; mkdir -p $O /tmp/sass
ncu --set full --import-source on --clock-control none -k regex:"k_warp" -c 1 -o /tmp/sass/kw python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu -i /tmp/sass/kw.ncu-rep --page source --csv --print-source sass > $O/kw_sass.csv 2> $O/kw.err
ncu --set full --import-source on --clock-control none -k regex:"k_extprod_cta" -c 1 -o /tmp/sass/ke python bench.py --extprod --steps 1 --warmup 1 > /dev/null 2>&1
ncu -i /tmp/sass/ke.ncu-rep --page source --csv --print-source sass > $O/ke_sass.csv 2> $O/ke.err
ncu -i /tmp/sass/ke.ncu-rep --page raw --csv > $O/ke_raw.csv 2>&1
ls -la $O
