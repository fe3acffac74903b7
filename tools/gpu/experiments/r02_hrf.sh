# HRF-MatVec launch shape sweep (unroll x j-split x min-blocks) + GPU tests of the round-2 changes
set -x
O=gpurun_out/r02f; mkdir -p $O
build() { RNT_NVCC_EXTRA="$1" python -c "from paper_2410_05934_b200 import build as b; b.build(force=True)" > /dev/null 2>&1; }
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
python bench.py --workload cfg2 --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_cfg2.json 2>&1
python bench.py --steps 30 --no-cpu-baseline --no-e2e --no-graph > $O/bench_cfg5.json 2>&1
python bench.py --extprod --steps 20 > $O/bench_extprod.json 2>&1
python bench.py --hrf --steps 10 > $O/bench_hrf_u2_js2_m1.json 2>&1
for cfg in "1 1 1" "1 2 1" "1 4 1" "2 1 4" "2 2 4" "2 4 4" "1 4 4" "2 2 3" "4 2 3" "1 8 1"; do
  set -- $cfg
  build "-DRNT_HRF_UNROLL=$1 -DRNT_HRF_JS=$2 -DRNT_HRF_MINB=$3"
  python bench.py --hrf --steps 10 > $O/bench_hrf_u$1_js$2_m$3.json 2>&1
done
build ""
grep -H '"results"' $O/bench_hrf*.json | python -c "
import json,sys
for ln in sys.stdin:
    f, j = ln.split(':', 1); d=json.loads(j); print(f.split('/')[-1], {k:(round(v['ms'],4), round(v['frac_hbm'],3)) for k,v in d['results'].items()})"
