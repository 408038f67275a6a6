python -c "from paper_2406_06022_b200 import build; build.build()" > /dev/null 2>&1
. scripts/summ.sh
GSB_AGG_W=128 timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/ag_w128.log 2>&1; summ gpurun_out/ag_w128.log 2>/dev/null | head -3
CMD="python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 1 --no-graph --pipeline off"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"agg_seg|agg_kernel" -s 2 -c 2 -o gpurun_out/agseg $CMD > gpurun_out/agseg_ncu.log 2>&1; echo ncu rc $?
GSB_AGG=warp timeout 600 ncu --set full --import-source on --clock-control none -k regex:"agg_seg|agg_kernel" -s 2 -c 2 -o gpurun_out/agwarp $CMD > gpurun_out/agwarp_ncu.log 2>&1; echo ncu rc $?
