CMD="python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 1 --no-graph"
for v in 1 0; do
GSB_AGG=$v timeout 300 $CMD > gpurun_out/agg2_plain$v.log 2>&1 && GSB_AGG=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:"agg" -s 4 -c 2 -o gpurun_out/agg2_v$v $CMD > gpurun_out/agg2_ncu$v.log 2>&1; echo rc $?
done
