# agg_kernel dynamic row scheduler: parity + bench A/B (mag bf16 / f32, amazon_lp) against the static stride
cp scripts/libgsb_dyn.bin paper_2406_06022_b200/libgsb.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/dy_tests.log 2>&1; echo tests rc $?; tail -1 gpurun_out/dy_tests.log
for v in sta dyn sta dyn; do bash scripts/gpu_binab.sh dy agg "" $v; bash scripts/gpu_binab.sh dy agg "--feat-dtype f32" $v; done
for v in sta dyn; do bash scripts/gpu_binab.sh dy agg_l0 "--config amazon_lp" $v; done
