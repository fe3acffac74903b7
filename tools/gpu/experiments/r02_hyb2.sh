O=gpurun_out/hyb2; mkdir -p $O
for c in 2 4; do ./tools/microbench/hyb $c; done > $O/hyb.jsonl 2>&1
cat $O/hyb.jsonl | grep -v '"cta_per_sm":2,' | sort -u
ncu --clock-control none -k regex:"k_chain<6|k_chain<7" --metrics regex:sm__inst_executed_pipe_.*.avg.pct_of_peak_sustained_active,regex:sm__pipe_.*_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,regex:smsp__average_warp_latency_issue_stalled.*.ratio --csv ./tools/microbench/hyb 4 > $O/hyb_ncu.csv 2> $O/hyb_ncu.err
