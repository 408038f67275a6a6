for e in GSB_DWC_SIDE=0 GSB_DWC_SIDE=1 GSB_DWC_SIDE=0 GSB_DWC_SIDE=1; do
  env $e timeout 300 python bench.py --config gcn_1b --no-cpu-baseline > gpurun_out/e2_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/e2_b.log').read().strip().splitlines()[-1]); print('$e', round(l['ms_per_step'],4), round(l['value']/1e6,3), round(l['e2e']['value']/1e6,3))"
done
