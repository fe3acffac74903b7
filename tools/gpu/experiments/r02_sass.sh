# per-SASS-instruction execution counts of the dominant kernels (ncu source page)
O=gpurun_out/sass; mkdir -p $O /tmp/sass
ncu --set full --import-source on --clock-control none -k regex:"k_warp" -c 1 -o /tmp/sass/kw python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_row|k_col" -c 3 -o /tmp/sass/k16 python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu -i /tmp/sass/kw.ncu-rep --page source --csv --print-source sass > $O/kw_sass.csv 2> $O/kw.err
ncu -i /tmp/sass/k16.ncu-rep --page source --csv --print-source sass > $O/k16_sass.csv 2> $O/k16.err
ls -la $O; head -3 $O/kw_sass.csv
