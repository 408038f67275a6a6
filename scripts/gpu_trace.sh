python -c "from paper_2406_06022_b200 import build; build.build()" > /dev/null 2>&1
for d in 1024 1031; do GSB_GEMM_DBG=$d timeout 60 python scripts/gemm_trace.py; done
M=16384 GSB_GEMM_DBG=1024 timeout 60 python scripts/gemm_trace.py
for d in 0 1; do GSB_GEMM_DBG=$d timeout 120 python scripts/gemm_micro.py; done
GSB_GEMM=umma timeout 120 python scripts/gemm_micro.py
