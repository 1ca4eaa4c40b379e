#!/bin/bash
# iteration: GPU tests (fast subset unless FULL=1), bench, launch list + one full ncu capture
mkdir -p gpurun_out
python scripts/write_bw.py > gpurun_out/write_bw.json 2>&1
if [ "${FULL:-0}" = "1" ]; then SEL=""; else SEL="-k not full_size_sampled"; fi
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 "$SEL" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 2 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench.log
if [ "${PROF:-1}" = "1" ]; then
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"count_kernel|write_kernel" -s 8 -c 4 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
fi
