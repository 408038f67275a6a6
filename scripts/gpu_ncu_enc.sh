# ncu --set full of the input-encoder kernels on the MAG240M-shaped 1/16 config (eager step)
T=${1:-ncue}
mkdir -p gpurun_out
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
CMD="python bench.py --config mag240m_1_16 --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 1 --no-graph --pipeline off"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1; echo plain rc $?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"enc_umma|tma3_gemm" -s 6 -c 6 -o gpurun_out/${T} $CMD > gpurun_out/${T}_ncu.log 2>&1; echo ncu rc $?
ncu -i gpurun_out/${T}.ncu-rep --page details --csv > gpurun_out/${T}_details.csv 2>/dev/null; echo done
