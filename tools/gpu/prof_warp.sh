ncu --set full --clock-control none --import-source on -k regex:k_warp -s 2 -c 1 -o gpurun_out/prof_warp2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_warp.log 2>&1
tail -3 gpurun_out/ncu_full_warp.log
