nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -30
