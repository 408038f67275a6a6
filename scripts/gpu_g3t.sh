# per-role timeline + knob sweep of the tma3 GEMM (NN, M=1024 and 16384)
T=$1
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
for d in 1024 1031 1039 1536 1543; do for m in 1024 16384; do M=$m GSB_GEMM_DBG=$d timeout 60 python scripts/gemm_trace.py 2>&1; done; done
for d in 0 512; do GSB_GEMM_DBG=$d timeout 120 python scripts/gemm_micro.py 2>&1 | grep "mode=" ; done
