# key switch (f2): k_row_mac occupancy / prefetch / digit split; ncu of k_row_mac and k_extprod_cta
set -x
O=gpurun_out/r02i; mkdir -p $O /tmp/r02i
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1; }
python bench.py --keyswitch --steps 10 > $O/bench_ks.json 2>&1
ncu --set full --clock-control none -k regex:"k_row_mac|k_col_fwd" -c 2 -o /tmp/r02i/ks python bench.py --keyswitch --steps 1 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_extprod_cta" -c 1 -o /tmp/r02i/ext python bench.py --extprod --steps 1 --warmup 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_ks /tmp/r02i/ks.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py $O/ncu_extprod /tmp/r02i/ext.ncu-rep > /dev/null 2>&1
for v in "-DRNT_ROWMAC_MINB=3" "-DRNT_ROWMAC_PREFETCH=1" "-DRNT_ROWMAC_PREFETCH=1 -DRNT_ROWMAC_MINB=1" "-DRNT_KS_SPLIT=2" "-DRNT_KS_SPLIT=3"; do
  build "$v"; n=$(echo "$v" | tr -d ' =-' | tr 'A-Z' 'a-z')
  python bench.py --keyswitch --steps 10 > $O/bench_ks_$n.json 2>&1
done
build ""
grep -H '"results"' $O/bench_ks*.json | python -c "
import json,sys
for ln in sys.stdin:
    f, j = ln.split(':', 1); d=json.loads(j); print(f.split('/')[-1], {k:round(v['ms'],4) for k,v in d['results'].items()})"
cat $O/ncu_ks.md $O/ncu_extprod.md
