summ() { python - "$1" <<'PY'
import json, sys
l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', round(l['value']), l['unit'], 'ms/step', round(l['ms_per_step'], 4), 'e2e', round(l['e2e']['value']),
      'roof', (l.get('roofline') or {}).get('kernel'), round((l.get('roofline') or {}).get('frac', 0), 3))
for k, v in list(l['kernels'].items())[:5]: print(f'   {k:22s} {v["us_per_step"]:8.1f}')
PY
}
for N in 2 4; do for G in unique fused; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2964$N bench.py --gpus $N --peer-gather $G --steps 150 > gpurun_out/b29_${N}_${G}.log 2> gpurun_out/b29_${N}_${G}.err; echo $N $G rc $?; summ gpurun_out/b29_${N}_${G}.log
done; done
