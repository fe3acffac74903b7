# verify HEAD: GPU tests, smoke, default bench line, 2 shared ranks
O=gpurun_out/head; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
python __graft_entry__.py --smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py --steps 50 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "bench rc=$?"
tail -1 $O/bench_cfg5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['digests_ok'], d['clocks'], d['gpu_launches'], d['cpu_baseline']['value'])"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; tail -1 $O/bench_reference.json | head -c 300; echo
RNT_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_share2.json 2> $O/bench_share2.err; echo "share2 rc=$?"
