CMD="python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 1 --no-graph"
for v in 2; do
GSB_AGG=$v timeout 300 $CMD > gpurun_out/agg5_plain$v.log 2>&1 && GSB_AGG=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:"agg" -s 4 -c 1 -o gpurun_out/agg5_v$v $CMD > gpurun_out/agg5_ncu$v.log 2>&1; echo rc $?
done
