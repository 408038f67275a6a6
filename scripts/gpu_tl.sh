# full GPU suite (no -x) + one per-launch timeline of the mag step
T=$1
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -4 gpurun_out/${T}_tests.log
GSB_TIMELINE=gpurun_out/${T}_timeline.txt timeout 300 python bench.py --steps 100 --no-cpu-baseline --profile-steps 1 > gpurun_out/${T}_b.log 2>&1; echo bench rc $?
python scripts/timeline.py gpurun_out/${T}_timeline.txt > gpurun_out/${T}_timeline_view.txt; head -80 gpurun_out/${T}_timeline_view.txt
