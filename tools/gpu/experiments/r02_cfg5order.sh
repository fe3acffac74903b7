# cfg5 part order and 2^16 limb-window count (RNT_EXPERIMENTS build)
O=gpurun_out/order; mkdir -p $O
for g in 2 1 3; do for rev in "" "--reverse-parts"; do
  RNT_SPLIT_G=$g python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-graph $rev > $O/b_g${g}${rev}.json 2>&1
  echo "split_g=$g $rev $(tail -1 $O/b_g${g}${rev}.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["value"]/1e6,2))')"
done; done
for g in 2 1 3 4; do RNT_SPLIT_G=$g python bench.py --workload cfg3 --steps 50 --no-cpu-baseline --no-e2e --no-graph > $O/c3_g$g.json 2>&1; echo "cfg3 split_g=$g $(tail -1 $O/c3_g$g.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4))')"; done
