#!/bin/bash
# GPU parity (all -m gpu tests) + bench in the given modes (MODES, default records full)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for m in ${MODES:-records full}; do
  timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode $m > gpurun_out/bench_$m.log 2>&1
  echo "$m :: $(python3 -c "
import json; d=json.loads(open('gpurun_out/bench_$m.log').read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()}, '%.0f'%(d['roofline']['achieved'] or 0))" 2>&1 | tail -1)"
done
