# cluster single-launch path (RNT_CLUSTER_UNITS hook) for the 8-GPU 2^16 shards (22-23 limbs)
O=gpurun_out/clu; mkdir -p $O
for cu in 2 64; do
  for L in 23 12 45; do
    RNT_CLUSTER_UNITS=$cu python bench.py --log2n 16 --limbs $L --batch 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > $O/cu${cu}_L$L.json 2>&1
    echo "cluster_units=$cu L=$L $(tail -1 $O/cu${cu}_L$L.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')"
  done
done
