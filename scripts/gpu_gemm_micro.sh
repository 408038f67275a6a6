mkdir -p gpurun_out
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/gm_build.log 2>&1
for d in ${DBGS:-0 7 15 23 31 8 16 24}; do GSB_GEMM_DBG=$d timeout 120 python scripts/gemm_micro.py; done
