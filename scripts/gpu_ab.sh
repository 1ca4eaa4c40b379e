#!/bin/bash
# parity tests (default pipeline) + bench A/B over env variants (VARIANTS) and modes (MODES)
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
for v in ${VARIANTS:-"ME_PIPE=2"}; do
  for m in ${MODES:-records}; do
  env $(echo $v | tr , " ") timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode $m > gpurun_out/bench_ab.log 2>&1
  echo "$v $m :: $(python3 -c "
import json; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()}, '%.0f'%(d['roofline']['achieved'] or 0) if d.get('roofline') else '')" 2>&1 | tail -1)"
  done
done
