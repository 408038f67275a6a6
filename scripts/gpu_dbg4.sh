python -c "from paper_2406_06022_b200 import build; build.build()" > /dev/null 2>&1
CUDA_LAUNCH_BLOCKING=1 GSB_DEBUG_SYNC=1 timeout 600 python -m pytest tests/test_gpu_partitioned.py -x -q -k mag_small 2>&1 | grep -E "Error|error|gsb|failed|passed" | head -30
