# e2e chunking sweep (ramped vs uniform chunks, chunk size).
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "execute_host" 2>&1 | tail -1
for r in 1 0; do for mb in 8 16 32; do
  RNT_CHUNK_RAMP=$r RNT_CHUNK_MB=$mb python bench.py --steps 20 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ramp $r mb $mb e2e %.3e value %.3e'%(d['e2e']['value'], d['value']))"
done; done
