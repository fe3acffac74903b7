nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/bv tools/microbench/bfly_variants.cu 2>/dev/null
/tmp/bv 2>&1 | grep -E "V0_nvcc|V14" | tail -2
ncu --metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:"k_bfly<(0|14)>" -c 4 /tmp/bv 2>/dev/null | grep -E "k_bfly|fmaheavy|alu|issue" | head -16
