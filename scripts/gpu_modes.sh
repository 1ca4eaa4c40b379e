#!/bin/bash
# bench the three output modes + ncu of the count and write kernels
mkdir -p gpurun_out
for m in count index full; do
  timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode $m > gpurun_out/bench_$m.log 2>&1
  echo "$m :: $(python3 -c "
import json; d=json.loads(open('gpurun_out/bench_$m.log').read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()})" 2>&1 | tail -1)"
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"count_kernel|write_kernel" -s 40 -c 4 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
