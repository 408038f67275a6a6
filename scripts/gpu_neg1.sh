timeout 900 python -m pytest tests/test_gpu_negatives.py tests/test_gpu_lp.py -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed|mismatch" | head -20
