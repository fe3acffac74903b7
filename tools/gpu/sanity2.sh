for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/gpu/sanitize.py 2>&1 | tail -3
done
echo "== torchrun nproc 1"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 --scaling strong --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-200
