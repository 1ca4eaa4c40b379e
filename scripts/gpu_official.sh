#!/bin/bash
# full GPU test suite, official bench line, launch list and one ncu capture of one chunk
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
python scripts/profile_chunk.py 40 > gpurun_out/chunk40.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"row_kernel|stage_kernel|scan_kernel|expand_kernel" -c 4 -o gpurun_out/prof python scripts/profile_chunk.py 40 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"; cat gpurun_out/chunk40.json
