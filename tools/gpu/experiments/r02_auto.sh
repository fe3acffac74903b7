O=gpurun_out/auto; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "automorph or hrot or keyswitch" > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
python bench.py --automorph --steps 20 > $O/bench_automorph.json 2>&1; tail -1 $O/bench_automorph.json
