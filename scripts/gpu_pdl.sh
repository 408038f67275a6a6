timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -5
for cfg in mag synth_1b amazon_lp mag240m_1_16; do
for np in 1 0; do
  GSB_NO_PDL=$np timeout 600 python bench.py --no-cpu-baseline --config $cfg --steps 200 > gpurun_out/pdl_${cfg}_$np.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/pdl_${cfg}_$np.log').read().strip().splitlines()[-1]); print('$cfg nopdl=$np', d['value'], d['ms_per_step'], d['e2e']['value'])"
done; done
