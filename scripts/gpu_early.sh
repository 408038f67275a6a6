timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -5
for cfg in mag synth_1b amazon_lp mag240m_1_16; do
  timeout 600 python bench.py --no-cpu-baseline --config $cfg --steps 200 > gpurun_out/early_${cfg}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/early_${cfg}.log').read().strip().splitlines()[-1]); print('$cfg', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
done
