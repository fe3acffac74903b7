# cfg2 / cfg5 with one warp per polynomial at 28 / 32 warps per SM (experiment builds in exp/)
O=gpurun_out/t1; mkdir -p $O
for v in base t1m14 t1m16; do
  cp exp/lib_$v.so paper_2410_05934_b200/librnsntt.so
  for w in cfg2 cfg5; do
    python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${v}_$w.json 2>&1
    echo "$v $w $(tail -1 $O/${v}_$w.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), [round(p["ms"],5) for p in d["parts"]], round(d["roofline"]["frac"],4))')"
  done
done
for b in 2048 3000 4144 6000 8192; do for v in base t1m14; do cp exp/lib_$v.so paper_2410_05934_b200/librnsntt.so
  python bench.py --log2n 10 --limbs 1 --batch $b --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${v}_b$b.json 2>&1
  echo "$v batch=$b $(tail -1 $O/${v}_b$b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), round(d["roofline"]["frac"],4))')"
done; done
cp exp/lib_base.so paper_2410_05934_b200/librnsntt.so
