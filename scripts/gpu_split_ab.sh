# splitter-warp count A/B (prebuilt exp/libgsb_sW.so) + tests of the current tree.  usage: bash scripts/gpu_split_ab.sh TAG
T=${1:-sab}
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py tests/test_gpu_fullscale.py tests/test_gpu_partition_sim.py tests/test_gpu_lp.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/${T}_tests.log
. scripts/summ.sh
cp paper_2406_06022_b200/libgsb.so /tmp/libgsb_cur.so
for v in s8 s4 s16; do
  cp exp/libgsb_$v.so paper_2406_06022_b200/libgsb.so
  for k in 1 2; do
    timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/${T}_bench_${v}_$k.log 2>&1
    python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_bench_${v}_$k.log').read().strip().splitlines()[-1]); print('$v', $k, round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'gemm_fwd_l0' in k or 'nc_' in k or 'scatter' in k or 'relu' in k})"
  done
done
cp /tmp/libgsb_cur.so paper_2406_06022_b200/libgsb.so
timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/${T}_bench_cur.log 2>&1
python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_bench_cur.log').read().strip().splitlines()[-1]); print('cur', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'gemm' in k or 'nc_' in k or 'scatter' in k or 'relu' in k or 'tcsr' in k})"
