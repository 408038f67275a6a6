timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed|mismatch" | head -30
