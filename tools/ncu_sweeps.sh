#!/bin/bash
# Full ncu capture of the live fp32 sweep kernels at the bench size (one GPU).
# usage: bash tools/ncu_sweeps.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_row_shift --launch-skip 1 -c 1 \
  -o gpurun_out/row_$TAG -f python tools/profile_sweeps.py 65536 > gpurun_out/ncu_row_$TAG.log 2>&1; echo "row rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_col_fast -c 1 \
  -o gpurun_out/col_$TAG -f python tools/profile_sweeps.py 65536 > gpurun_out/ncu_col_$TAG.log 2>&1; echo "col rc=$?"
