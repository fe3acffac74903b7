ncu --set full --clock-control none --import-source on -k regex:"k_warp" -s 2 -c 1 -o gpurun_out/prof_kwarp_km3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/prof_kwarp_km3.ncu-rep --page source --csv --print-source sass > gpurun_out/src_kwarp_km3.csv 2>/dev/null
ls -la gpurun_out/ | head
