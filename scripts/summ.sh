# summ LOG : one-line summary of a bench.py JSON line + top kernels
summ() { python - "$1" <<'PY'
import json, sys
try:
    l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], 'no JSON', e); sys.exit(0)
print(sys.argv[1], 'value', round(l['value']), l['unit'], 'ms/step', round(l['ms_per_step'], 4), 'e2e', round(l['e2e']['value']),
      'roof', (l.get('roofline') or {}).get('kernel'), round((l.get('roofline') or {}).get('frac', 0), 3), 'clk', l.get('clocks'),
      'launches', l.get('gpu_launches'))
for k, v in list(l['kernels'].items())[:5]: print(f'   {k:22s} {v["us_per_step"]:8.1f}')
PY
}
