#!/bin/bash
# launch list + one full ncu capture of the sweep kernels (bench's own launch configuration)
mkdir -p gpurun_out
python scripts/write_bw.py > gpurun_out/write_bw.json 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"count_kernel|write_kernel" -s 8 -c 4 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -2 gpurun_out/plain.log gpurun_out/ncu_full.log
