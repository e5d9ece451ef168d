#!/bin/bash
# single-pass vs two-pass at cfg3: ms/step and the in-solve kernel split
# usage: tools/sp_cmp.sh "ENV=.. ENV2=.." "ENV=.." ...
[ -n "$SP_PARITY" ] && python -m pytest tests/test_gpu_parity.py -q -x -k fused 2>&1 | tail -3
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg OTG_VERBOSE=1 timeout 300 python bench.py --no-tol --no-cpu --steps 20 --warmup 3 > gpurun_out/sp_$$.log 2>&1
  grep "single-pass" gpurun_out/sp_$$.log | head -1
  grep '^{' gpurun_out/sp_$$.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = d['roofline']; print('ms/step', round(d['ms_per_step'], 3), 'row', round(r['row_pass_ms'], 3), 'col', round(r['col_pass_ms'], 3))
" || tail -5 gpurun_out/sp_$$.log
done
rm -f gpurun_out/sp_$$.log
