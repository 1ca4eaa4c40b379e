#!/bin/bash
# GPU tests (fast subset) + bench variants of the write pass
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -k "not full_size_sampled and not multi_gpu" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
ME_WRITE_BULK=0 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "small_spaces or subranges or caller" > gpurun_out/pytest_gpu0.log 2>&1; echo "pytest stage0 rc=$?"; tail -1 gpurun_out/pytest_gpu0.log
for v in ${VARIANTS:-"ME_GRID_MODE=1"}; do
  env $v timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_var.log 2>&1
  echo "$v :: $(python3 -c "
import json; d=json.loads(open('gpurun_out/bench_var.log').read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()}, '%.0f'%d['roofline']['achieved'])" 2>&1 | tail -1)"
done
for m in count index; do
  timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode $m > gpurun_out/bench_$m.log 2>&1
  echo "$m :: $(python3 -c "
import json; d=json.loads(open('gpurun_out/bench_$m.log').read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()})" 2>&1 | tail -1)"
done
