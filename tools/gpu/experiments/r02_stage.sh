# k_warp MODE 2 with the polynomials cp.async-staged into shared memory before the first pass
O=gpurun_out/stage; mkdir -p $O
for r in 1 2; do for v in base stage; do
  cp exp/lib_$v.so paper_2410_05934_b200/librnsntt.so
  line="$v run$r:"
  for b in 2368 2731 4096 16384; do
    python bench.py --log2n 10 --limbs 1 --batch $b --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${v}_b${b}_$r.json 2>&1
    line="$line $b:$(tail -1 $O/${v}_b${b}_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
  done
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${v}_cfg5_$r.json 2>&1
  echo "$line cfg5:$(tail -1 $O/${v}_cfg5_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1), d["digests_ok"])')"
done; done
cp exp/lib_base.so paper_2410_05934_b200/librnsntt.so
