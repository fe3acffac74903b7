O=gpurun_out/e2e2; mkdir -p $O
for w in cfg5 cfg2 cfg3 cfg4; do
for cfg in "16 0" "32 1" "64 1" "128 1" "32 0"; do
  set -- $cfg
  if [ "$2" = "1" ]; then export RNT_E2E_NORAMP=1; else unset RNT_E2E_NORAMP; fi
  st=20; [ $w = cfg4 ] && st=10
  RNT_E2E_CHUNK_MB=$1 python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-graph > $O/b_${w}_$1_$2.json 2>&1
  echo "$w chunk=$1MB noramp=$2 $(tail -1 $O/b_${w}_$1_$2.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["value"]/1e6,4))')"
done; done
unset RNT_E2E_NORAMP
RNT_E2E_CHUNK_MB=32 RNT_E2E_NORAMP=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-graph --e2e-serial > $O/b_serial_32_1.json 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-graph --e2e-serial > $O/b_serial_16_0.json 2>&1
for f in $O/b_serial*; do echo $f $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["value"]/1e6,4))'); done
