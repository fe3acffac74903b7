# N=2^10 polymul: 2-warp teams (16 CTAs/SM) vs 4-warp teams (8 CTAs/SM) across batch sizes
O=gpurun_out/t4; mkdir -p $O
for v in base t4; do
  cp exp/lib_$v.so paper_2410_05934_b200/librnsntt.so
  line="$v:"
  for b in 1200 2368 2731 3000 3552 4096 6000 8192 16384; do
    python bench.py --log2n 10 --limbs 1 --batch $b --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${v}_b$b.json 2>&1
    line="$line $b:$(tail -1 $O/${v}_b$b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
  done
  echo "$line"
done
cp exp/lib_base.so paper_2410_05934_b200/librnsntt.so
