nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/bv tools/microbench/bfly_variants.cu 2>/dev/null
/tmp/bv | tail -6
ncu --clock-control none --metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:k_bfly -c 6 --csv /tmp/bv 2>/dev/null | grep -E "k_bfly" | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/"//g' | tail -18
