nvidia-smi --query-gpu=index,name --format=csv
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu --tb=short 2>&1 | tail -15
