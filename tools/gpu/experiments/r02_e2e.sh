# e2e chunking sweep on an RNT_EXPERIMENTS build + automorph tests/bench on the same build
O=gpurun_out/e2e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "automorph or hrot or keyswitch or bconv or execute" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
python bench.py --automorph --steps 20 > $O/bench_automorph.json 2>&1; tail -1 $O/bench_automorph.json
for cfg in "16 0" "8 0" "32 0" "64 0" "16 1" "32 1" "4 1"; do
  set -- $cfg
  if [ "$2" = "1" ]; then export RNT_E2E_NORAMP=1; else unset RNT_E2E_NORAMP; fi
  RNT_E2E_CHUNK_MB=$1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-graph > $O/b_$1_$2.json 2>&1
  echo "chunk=$1MB noramp=$2 $(tail -1 $O/b_$1_$2.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["value"]/1e6,3), round(d["value"]/1e6,2))')"
done
unset RNT_E2E_NORAMP
for w in cfg2 cfg3; do for c in 16 4; do RNT_E2E_CHUNK_MB=$c python bench.py --workload $w --steps 20 --no-cpu-baseline --no-graph > $O/b_${w}_$c.json 2>&1; echo "$w chunk=$c $(tail -1 $O/b_${w}_$c.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["value"]/1e6,3))')"; done; done
