# k_warp L2 prefetch variants (exp/lib_pf{0,1,2}.so)
O=gpurun_out/pf; mkdir -p $O
for r in 1 2; do for v in 0 1 2; do
  cp exp/lib_pf$v.so paper_2410_05934_b200/librnsntt.so
  python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/cfg5_pf${v}_$r.json 2>&1
  python bench.py --workload cfg2 --steps 50 --no-cpu-baseline --no-e2e --no-graph > $O/cfg2_pf${v}_$r.json 2>&1
  echo "pf$v run$r cfg5 $(tail -1 $O/cfg5_pf${v}_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), [round(p["ms"],5) for p in d["parts"]], d["digests_ok"])') cfg2 $(tail -1 $O/cfg2_pf${v}_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), d["digests_ok"])')"
done; done
cp exp/lib_pf0.so paper_2410_05934_b200/librnsntt.so
