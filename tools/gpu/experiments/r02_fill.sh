# strong-scaling planner "fill" (coarse parts on whole ranks, the 2^10 batch filling every rank) vs "parts"
O=gpurun_out/fill; mkdir -p $O
for pl in fill parts; do for n in 4 8; do
  line="$pl N=$n:"
  for r in $(seq 0 $((n-1))); do
    python bench.py --gpus $n --emulate-rank $r --shard $pl --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${pl}_${n}_$r.json 2>&1
    line="$line $(tail -1 $O/${pl}_${n}_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
  done
  echo "$line"
done; done
