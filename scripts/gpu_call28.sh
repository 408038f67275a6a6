summ() { python - "$1" <<'PY'
import json, sys
l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', round(l['value']), l['unit'], 'ms/step', round(l['ms_per_step'], 4), 'e2e', round(l['e2e']['value']),
      'roof', (l.get('roofline') or {}).get('kernel'), round((l.get('roofline') or {}).get('frac', 0), 3), 'clk', l.get('clocks'))
for k, v in list(l['kernels'].items())[:5]: print(f'   {k:22s} {v["us_per_step"]:8.1f}')
PY
}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|passed|failed" | head -20
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b28_mag1.log 2> gpurun_out/b28_mag1.err; echo mag1 rc $?; summ gpurun_out/b28_mag1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 4 > gpurun_out/b28_mag4.log 2> gpurun_out/b28_mag4.err; echo mag4 rc $?; summ gpurun_out/b28_mag4.log; tail -2 gpurun_out/b28_mag4.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 > gpurun_out/b28_mag2.log 2> gpurun_out/b28_mag2.err; echo mag2 rc $?; summ gpurun_out/b28_mag2.log
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 4 --config synth_1b --steps 100 > gpurun_out/b28_1b4.log 2> gpurun_out/b28_1b4.err; echo 1b4 rc $?; summ gpurun_out/b28_1b4.log; tail -2 gpurun_out/b28_1b4.err
