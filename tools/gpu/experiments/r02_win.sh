# limb windows for single-polynomial 2^16 polymuls of 12 / 23 / 45 limbs (RNT_EXPERIMENTS build)
O=gpurun_out/win; mkdir -p $O
cp exp/lib_exp.so paper_2410_05934_b200/librnsntt.so
for L in 12 23 45; do
  line="L=$L:"
  for g in 1 2 3 4; do
    RNT_SPLIT_G=$g python bench.py --log2n 16 --limbs $L --batch 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/L${L}_g$g.json 2>&1
    line="$line g$g:$(tail -1 $O/L${L}_g$g.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
  done
  echo "$line"
done
cp exp/lib_base.so paper_2410_05934_b200/librnsntt.so
