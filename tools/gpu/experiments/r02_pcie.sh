O=gpurun_out/pcie; mkdir -p $O
nvidia-smi -q | grep -iA3 "PCIe Generation\|Link Width" > $O/link.txt 2>&1
python tools/gpu/pcie_bw.py > $O/pcie.json 2>&1; cat $O/pcie.json; cat $O/link.txt | head -20
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2>&1; tail -1 $O/bench_cfg5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
