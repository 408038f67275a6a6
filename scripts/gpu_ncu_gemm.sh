# ncu --set full of the TMA GEMM kernels (one bench step, eager).  usage: bash scripts/gpu_ncu_gemm.sh TAG [regex]
T=${1:-ncug}; R=${2:-tma_gemm}
mkdir -p gpurun_out
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
CMD="python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 1 --no-graph --pipeline off"
timeout 300 $CMD > gpurun_out/${T}_plain.log 2>&1; echo plain rc $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$R" -s 10 -c 8 -o gpurun_out/${T} $CMD > gpurun_out/${T}_ncu.log 2>&1; echo ncu rc $?
ncu -i gpurun_out/${T}.ncu-rep --page details --csv > gpurun_out/${T}_details.csv 2>/dev/null; echo done
