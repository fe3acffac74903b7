O=gpurun_out/frac; mkdir -p $O
for f in 0 60 67 75 40 33; do
  RNT_SPLIT_FRAC=$f python bench.py --workload cfg3 --steps 50 --no-cpu-baseline --no-e2e --no-graph > $O/c3_$f.json 2>&1
  RNT_SPLIT_FRAC=$f python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/c5_$f.json 2>&1
  echo "frac=$f cfg3 $(tail -1 $O/c3_$f.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), d["digests_ok"])') cfg5 $(tail -1 $O/c5_$f.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), d["digests_ok"])')"
done
