#!/bin/bash
# per-launch kernel times of one C5 chunk (ncu launch list; cold, serialised)
mkdir -p gpurun_out
python scripts/profile_chunk.py 40 ${PMODE:-records} > gpurun_out/chunk40.json 2>&1 || { cat gpurun_out/chunk40.json; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chunk_launches.csv \
  python scripts/profile_chunk.py 40 ${PMODE:-records} > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python3 scripts/launch_summary.py gpurun_out/chunk_launches.csv | tail -12
