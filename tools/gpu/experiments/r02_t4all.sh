O=gpurun_out/t4all; mkdir -p $O
for r in 1 2; do for v in base t4all; do
  cp exp/lib_$v.so paper_2410_05934_b200/librnsntt.so
  python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${v}_$r.json 2>&1
  echo "$v run$r cfg5: $(tail -1 $O/${v}_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1), [round(p["ms"]*1000,1) for p in d["parts"]], d["digests_ok"])')"
done; done
cp exp/lib_base.so paper_2410_05934_b200/librnsntt.so
