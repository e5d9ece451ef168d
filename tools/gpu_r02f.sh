#!/bin/bash
# Round-2 GPU pass: GPU tests, smoke, cfg3 bench, cfg5 bench, launch list of
# the cfg3 bench steady state (ncu, timing only, caches not flushed).
# Usage: tools/gpu_r02f.sh TAG
set -u
mkdir -p gpurun_out
TAG=${1:-r02f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/gputests_$TAG.log 2>&1; echo "gpu tests rc=$?"
tail -2 gpurun_out/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_$TAG.json | cut -c1-200
timeout 900 python bench.py --config 5 --steps 100 --warmup 3 > gpurun_out/bench5_$TAG.json 2> gpurun_out/bench5_$TAG.err; echo "bench5 rc=$?"
tail -1 gpurun_out/bench5_$TAG.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-tol --no-cpu \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
