#!/bin/bash
# N=1 C5 bench under launch-knob variants (kernel-only legs)
mkdir -p gpurun_out
for V in "" "ME_EXPAND_BPS=3" "ME_ROWS_SPAN=8" "ME_ROWS_SPAN=12" "ME_SETS=3" "ME_EXPAND_BPS=3 ME_ROWS_SPAN=8" ""; do
  env $V timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/knob.log 2>&1
  echo "[$V] rc=$? $(tail -1 gpurun_out/knob.log | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(round(d["ms_per_step"],1), "%.3e"%d["value"], d["feasible_per_step"])')"
done
