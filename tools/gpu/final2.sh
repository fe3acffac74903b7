set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -3
python __graft_entry__.py --smoke 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/final_cfg5.json
python -c "import json; d=json.load(open('gpurun_out/final_cfg5.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['step_frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'], d['gpu_launches'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-300
