O=gpurun_out/hyb3; mkdir -p $O
./tools/microbench/hyb 4 > $O/hyb.jsonl 2>&1; sort -u $O/hyb.jsonl
ncu --clock-control none --metrics regex:sm__inst_executed_pipe_.*.avg.pct_of_peak_sustained_active,regex:sm__pipe_.*_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,regex:smsp__average_warp_latency_issue_stalled.*.ratio --csv ./tools/microbench/hyb 4 > $O/hyb_ncu.csv 2> $O/hyb_ncu.err
