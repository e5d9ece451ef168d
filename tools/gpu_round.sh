#!/bin/bash
# One GPU round: GPU tests, bench line, launch list (ncu, timing only) and one
# full ncu capture of each sweep kernel at the bench size (steady-state launch).
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/gputests_$TAG.log 2>&1; echo "gpu tests rc=$?"
tail -2 gpurun_out/gputests_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_$TAG.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-tol --no-cpu \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function \
  -k regex:'^k_row_shift$' --launch-skip 1 -c 1 -o gpurun_out/row_$TAG -f \
  python tools/profile_sweeps.py 65536 > gpurun_out/ncu_row_$TAG.log 2>&1; echo "row full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function \
  -k regex:'^k_col_fast$' --launch-skip 1 -c 1 -o gpurun_out/col_$TAG -f \
  python tools/profile_sweeps.py 65536 > gpurun_out/ncu_col_$TAG.log 2>&1; echo "col full rc=$?"
