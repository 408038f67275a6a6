# round-2 evidence on one B200: GPU suite, smoke, bench lines (mag + cpu_baseline, reference arm,
# synth_1b, gcn_1b), NVTX-named ncu launch list with DRAM traffic, one ncu --set full capture,
# SASS instruction counts.  usage: bash scripts/gpu_r2_full.sh TAG
T=${1:-r2f}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/${T}_smoke.log
. scripts/summ.sh
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench rc $?; summ gpurun_out/${T}_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_ref.log 2>&1; echo ref rc $?; tail -c 300 gpurun_out/${T}_ref.log; echo
for c in synth_1b gcn_1b amazon_lp mag240m_1_16; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.log 2>&1; echo bench $c rc $?; summ gpurun_out/${T}_bench_$c.log | head -2
done
timeout 600 python bench.py --feat-dtype f32 --no-cpu-baseline > gpurun_out/${T}_bench_mag_f32.log 2>&1; echo bench mag f32 rc $?; summ gpurun_out/${T}_bench_mag_f32.log | head -2
GSB_LP_WARP=1 timeout 600 python bench.py --config amazon_lp --no-cpu-baseline > gpurun_out/${T}_bench_amazon_lp_warp.log 2>&1; echo bench lp warp rc $?; summ gpurun_out/${T}_bench_amazon_lp_warp.log | head -2
CMD="python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 2 --no-graph --pipeline off"
timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --print-units base --clock-control none --csv --log-file gpurun_out/${T}_traffic.csv $CMD > gpurun_out/${T}_ncu_traffic.log 2>&1; echo traffic rc $?
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --print-nvtx-rename kernel \
  -k regex:"agg_kernel|agg_quarter_kernel|agg_half_kernel|agg_seg_kernel|tma3_gemm_kernel|fill_kernel" -s 12 -c 6 -o gpurun_out/${T}_full $CMD > gpurun_out/${T}_ncu_full.log 2>&1; echo full rc $?
cuobjdump -sass paper_2406_06022_b200/libgsb.so > /tmp/sass.txt 2>/dev/null
for m in UTCHMMA UTCBAR UTMALDG UBLKCP LDTM LDG.E.ENL2.256 SYNCS; do echo "$m $(grep -c "$m" /tmp/sass.txt)"; done > gpurun_out/${T}_sass_counts.txt
grep -n "Function : \|UTMALDG\|UTCHMMA" /tmp/sass.txt | grep -B1 "UTMALDG\|UTCHMMA" | head -60 > gpurun_out/${T}_sass_excerpt.txt
cat gpurun_out/${T}_sass_counts.txt
