O=gpurun_out/ext; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "extprod or external" > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
python bench.py --extprod --steps 20 > $O/bench_extprod.json 2>&1; tail -1 $O/bench_extprod.json
