#!/bin/bash
# Round-2 final GPU pass: GPU tests, smoke, cfg3 bench (default + 100 steps),
# cfg5 bench, steady-state launch list (ncu timing only) and one full ncu
# capture of k_sweep1 at cfg3.   Usage: tools/gpu_r02g.sh TAG
set -u
mkdir -p gpurun_out
TAG=${1:-r02g}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/gputests_$TAG.log 2>&1; echo "gpu tests rc=$?"
tail -2 gpurun_out/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_$TAG.json | cut -c1-200
timeout 900 python bench.py --steps 100 --warmup 3 --no-cpu > gpurun_out/bench100_$TAG.json 2> gpurun_out/bench100_$TAG.err; echo "bench100 rc=$?"
timeout 900 python bench.py --config 5 --steps 200 --warmup 5 > gpurun_out/bench5_$TAG.json 2> gpurun_out/bench5_$TAG.err; echo "bench5 rc=$?"
tail -1 gpurun_out/bench5_$TAG.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/benchref_$TAG.json 2> gpurun_out/benchref_$TAG.err; echo "bench ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/sp_one.py 65536 65536 6 \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep1 --launch-skip 3 -c 1 \
  -o gpurun_out/sweep1_$TAG -f python tools/sp_one.py 65536 65536 6 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
