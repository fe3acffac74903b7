# latency engine (k_lat) vs warp engine (4-warp teams) crossover for small N = 2^10 batches
O=gpurun_out/lat; mkdir -p $O
for lu in 512 0; do
  line="lat_units=$lu:"
  for b in 64 128 256 384 512 768 1024; do
    RNT_LAT_UNITS=$lu python bench.py --log2n 10 --limbs 1 --batch $b --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/lu${lu}_b$b.json 2>&1
    line="$line $b:$(tail -1 $O/lu${lu}_b$b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
  done
  echo "$line"
done
