#!/bin/bash
# iteration: GPU tests (fast subset unless FULL=1), bench, launch list + one full ncu capture
mkdir -p gpurun_out
if [ "${FULL:-0}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
else
  timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -k "not full_size_sampled and not multi_gpu" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 2 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()}, d['roofline'])" 2>&1 | tail -2
if [ "${PROF:-1}" = "1" ]; then
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"count_kernel|write_kernel" -s 40 -c 4 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
fi
