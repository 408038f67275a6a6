timeout 900 python bench.py --no-cpu-baseline --config mag240m_1_16 --steps 100 --warmup 5 --profile-steps 3 --learnable-emb > gpurun_out/f1_emb.log 2>&1; echo rc $?
python -c "import json; d=json.loads(open('gpurun_out/f1_emb.log').read().strip().splitlines()[-1]); print('emb', d['value'], d['ms_per_step'], d['config'].get('featureless_inputs'), sorted(((round(v['us_per_step']),k) for k,v in d['kernels'].items()), reverse=True)[:8])"
timeout 600 python scripts/featcon_bench.py > gpurun_out/featcon.log 2>&1; echo rc $?; tail -2 gpurun_out/featcon.log
