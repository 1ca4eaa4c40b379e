#!/bin/bash
# GPU parity (sweep subset) + bench variants
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x --timeout 900 -k "sweep or rank or caller or subranges" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-"ME_WRITE_COMB=1" "ME_WRITE_COMB=0" "ME_WRITE_COMB=1,ME_SERIAL=1"}; do
  for m in ${MODES:-full index}; do
  env $(echo $v | tr , " ") timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode $m > gpurun_out/bench_var.log 2>&1
  echo "$v $m :: $(python3 -c "
import json; d=json.loads(open('gpurun_out/bench_var.log').read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()}, '%.0f'%(d['roofline']['achieved'] or 0))" 2>&1 | tail -1)"
  done
done
