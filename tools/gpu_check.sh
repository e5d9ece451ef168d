#!/bin/bash
# One gpurun session: tests, smoke, short bench.  Logs land in gpurun_out/.
set -u
mkdir -p gpurun_out
{ nvidia-smi; nproc; lscpu | grep "Model name"; free -g | head -2; } > gpurun_out/host.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
if [ "${BENCH:-1}" = "1" ]; then
  timeout 1200 python bench.py --steps ${STEPS:-20} --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench.log
fi
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/bench.log 2>/dev/null
