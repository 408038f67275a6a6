# round-2 GPU evidence: GPU suite, smoke, default bench, launch list.  usage: bash scripts/gpu_r2.sh TAG [extra pytest args]
T=${1:-r2}; shift
mkdir -p gpurun_out
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/${T}_smoke.log
timeout 600 python bench.py --steps 200 > gpurun_out/${T}_bench.log 2>&1; echo bench rc $?
. scripts/summ.sh; summ gpurun_out/${T}_bench.log
