set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 python __graft_entry__.py 2>&1 | tail -5 || true
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 600 2>&1 | tail -30
