#!/bin/bash
# Round-2 ncu evidence (one GPU): the launch list of a short bench run
# (timing metric only) and one full capture of the single-pass sweep at the
# bench size.  Run only after the same commands exit 0 without ncu.
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-tol --no-cpu \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep1 --launch-skip 1 -c 1 \
  -o gpurun_out/sweep1_$TAG -f python tools/sp_one.py 65536 65536 3 > gpurun_out/ncu_sweep1_$TAG.log 2>&1
echo "sweep1 full rc=$?"
