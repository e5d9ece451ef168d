#!/bin/bash
# Round-2 GPU pass: GPU tests (incl. config-scale parity + world-2 libotg),
# smoke, bench line.  Usage: tools/gpu_r02.sh TAG [pytest-args...]
set -u
mkdir -p gpurun_out
TAG=${1:-r02}
shift || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -s --durations=25 "$@" > gpurun_out/gputests_$TAG.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_$TAG.json | cut -c1-400
