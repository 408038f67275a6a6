summ() { python - "$1" <<'PY'
import json, sys
l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', round(l['value']), l['unit'], 'ms/step', round(l['ms_per_step'], 4), 'e2e', round(l['e2e']['value']),
      'roof', (l.get('roofline') or {}).get('kernel'), round((l.get('roofline') or {}).get('frac', 0), 3))
for k, v in list(l['kernels'].items())[:6]: print(f'   {k:22s} {v["us_per_step"]:8.1f}')
PY
}
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_lp.py tests/test_gpu_multi.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|passed|failed" | head -20
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b27_mag1.log 2> gpurun_out/b27_mag1.err; echo mag1 rc $?; summ gpurun_out/b27_mag1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 > gpurun_out/b27_mag2.log 2> gpurun_out/b27_mag2.err; echo mag2 rc $?; summ gpurun_out/b27_mag2.log; tail -3 gpurun_out/b27_mag2.err
timeout 400 python bench.py --config synth_1b --steps 100 --no-cpu-baseline > gpurun_out/b27_1b1.log 2> gpurun_out/b27_1b1.err; echo 1b1 rc $?; summ gpurun_out/b27_1b1.log; tail -3 gpurun_out/b27_1b1.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 2 --config synth_1b --steps 100 > gpurun_out/b27_1b2.log 2> gpurun_out/b27_1b2.err; echo 1b2 rc $?; summ gpurun_out/b27_1b2.log; tail -3 gpurun_out/b27_1b2.err
