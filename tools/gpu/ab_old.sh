# A/B: current tree vs tmp_ab/old (an older commit's sources), same box.
run() { for wl in cfg3 cfg4 cfg5; do python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>>$GRAFT_REPO_ROOT/gpurun_out/ab_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $wl ms %.4f'%d['ms_per_step'], d['clocks']['sm_mhz'])"; done; }
run new
(cd tmp_ab/old && python -m paper_2410_05934_b200.build --force > /dev/null && run old)
run new
RNT_SPLIT=0 run new_nosplit
