python -c "from paper_2406_06022_b200 import build; build.build()" > /dev/null 2>&1
GSB_DEBUG_SYNC=1 timeout 600 python -m pytest tests/test_gpu_partition_sim.py -x -q 2>&1 | grep -E "gsb\]|Error:|failed|passed|assert" | head -10
