# N = 2^16 chain occupancy: column kernels at 4 CTAs/SM (<= 64 registers), row kernel at 3 (<= 85)
set -x
O=gpurun_out/r02p; mkdir -p $O
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True, verbose=True)" > $O/build_$2.txt 2>&1; }
for v in "def:" "c4:-DRNT_COL_MINB=4" "r3:-DRNT_ROW_MINB=3" "c4r3:-DRNT_COL_MINB=4 -DRNT_ROW_MINB=3"; do
  n=${v%%:*}; f=${v#*:}
  build "$f" $n
  for w in cfg3 cfg4 cfg5; do python bench.py --workload $w --steps 40 --no-cpu-baseline --no-e2e --no-graph > $O/bench_${w}_$n.json 2>&1; done
done
build "" def2
grep -h -A3 "k_col_fwdILi16ELi16ELb0ELb1E\|k_rowILi16ELi2ELi16ELb1E\|k_col_invILi16ELi16E" $O/build_c4r3.txt | grep -E "Compiling|registers|spill"
python -c "
import json,glob
for f in sorted(glob.glob('$O/bench_cfg*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), [round(p['ms'],4) for p in d['parts']], d.get('digests_ok'))
"
