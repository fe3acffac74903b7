# strong-scaling shard planners: every rank's shard of cfg5 timed on one GPU (bench --emulate-rank)
O=gpurun_out/emul; mkdir -p $O
for pl in contig mixed; do for n in 2 4 8; do
  line="$pl N=$n:"
  for r in $(seq 0 $((n-1))); do
    python bench.py --gpus $n --emulate-rank $r --shard $pl --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/${pl}_${n}_$r.json 2>&1
    line="$line $(tail -1 $O/${pl}_${n}_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
  done
  echo "$line"
done; done
