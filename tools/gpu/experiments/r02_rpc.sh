# k_row with 8 rows (128 threads) per CTA at 4 CTAs/SM vs 16 rows at 2 CTAs/SM
O=gpurun_out/rpc; mkdir -p $O
for r in 1 2; do for v in base rpc8; do
  cp exp/lib_$v.so paper_2410_05934_b200/librnsntt.so
  line="$v run$r:"
  for w in cfg3 cfg5; do
    python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${v}_${w}_$r.json 2>&1
    line="$line $w:$(tail -1 $O/${v}_${w}_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1), d["digests_ok"])')"
  done
  python bench.py --log2n 16 --limbs 23 --batch 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${v}_L23_$r.json 2>&1
  echo "$line L23:$(tail -1 $O/${v}_L23_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
done; done
cp exp/lib_base.so paper_2410_05934_b200/librnsntt.so
