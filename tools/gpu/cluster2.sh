timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variants and env14" 2>&1 | grep -v "^  " | tail -30
