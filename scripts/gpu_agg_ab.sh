# A/B of the segment-parallel aggregation against the warp-per-row kernel (GSB_AGG=warp).  usage: bash scripts/gpu_agg_ab.sh TAG
T=${1:-aab}
mkdir -p gpurun_out
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py tests/test_gpu_inference.py tests/test_gpu_lp.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/${T}_tests.log
. scripts/summ.sh
for a in seg warp; do
  GSB_AGG=$a timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/${T}_bench_$a.log 2>&1; echo bench $a rc $?
  summ gpurun_out/${T}_bench_$a.log
done
