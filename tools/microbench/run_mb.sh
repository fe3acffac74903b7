set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/mb_clocks.csv &
SMI=$!
./tools/microbench/int_pipes | tee gpurun_out/int_pipes.jsonl
kill $SMI
lscpu | head -20 > gpurun_out/lscpu.txt
python -c 'import os; print(len(os.sched_getaffinity(0)))' >> gpurun_out/lscpu.txt
