# A/B of the TMA warp-specialized GEMM against the cp.async kernel (GSB_GEMM=umma).  usage: bash scripts/gpu_gemm_ab.sh TAG
T=${1:-gab}
mkdir -p gpurun_out
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q -k "gemm or nc_loss or nc_step or splitk or graph" > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/${T}_tests.log
. scripts/summ.sh
for g in tma umma; do
  GSB_GEMM=$g timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/${T}_bench_$g.log 2>&1; echo bench $g rc $?
  summ gpurun_out/${T}_bench_$g.log
done
