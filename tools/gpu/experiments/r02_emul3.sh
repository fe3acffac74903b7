# per-rank shard timings (parts planner) after the chain PDL change
O=gpurun_out/emul3; mkdir -p $O
for n in 2 4 8; do
  line="parts N=$n:"
  for r in $(seq 0 $((n-1))); do
    python bench.py --gpus $n --emulate-rank $r --shard parts --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/parts_${n}_$r.json 2>&1
    line="$line $(tail -1 $O/parts_${n}_$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
  done
  echo "$line"
done
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/one.json 2>&1; echo "N=1: $(tail -1 $O/one.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
