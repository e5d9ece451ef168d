#!/bin/bash
# GPU round + full ncu captures of the on-the-fly (cfg5-shaped) sweep kernels.
set -u
TAG=${1:-r01}
bash tools/gpu_round.sh $TAG
N=${OTF_N:-50000}
timeout 600 python tools/profile_otf.py $N > gpurun_out/otf_time_$TAG.log 2>&1; echo "otf time rc=$?"
cat gpurun_out/otf_time_$TAG.log | tail -2
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function \
  -k regex:'^k_row_shift$' --launch-skip 1 -c 1 -o gpurun_out/otfrow_$TAG -f \
  python tools/profile_otf.py $N > gpurun_out/ncu_otfrow_$TAG.log 2>&1; echo "otf row full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function \
  -k regex:'^k_col_fast$' --launch-skip 1 -c 1 -o gpurun_out/otfcol_$TAG -f \
  python tools/profile_otf.py $N > gpurun_out/ncu_otfcol_$TAG.log 2>&1; echo "otf col full rc=$?"
