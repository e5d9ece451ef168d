#!/bin/bash
# One GPU round: bench line, launch list (ncu, timing only) and one full
# ncu capture of the two sweep kernels at the bench size.
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-tol --no-cpu \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_(row_shift|col_fast)' -c 2 \
  -o gpurun_out/full_$TAG -f python tools/profile_sweeps.py 65536 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full rc=$?"
