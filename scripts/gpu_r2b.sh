#!/bin/bash
# round-2 GPU pass b: tests, default bench, launch list, ncu of chunk 40 (K0 rowcount + K3 fused)
O=gpurun_out/r2b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
ME_SERIAL=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-modes > $O/bench_serial.log 2>&1; echo "rc=$?" >> $O/bench_serial.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-modes > $O/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $O/ncu_launch.log
python scripts/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
python scripts/profile_chunk.py 40 records > $O/chunk40.json 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:rowcount_kernel|fused_kernel|scan_kernel" -c 3 \
  -o $O/prof python scripts/profile_chunk.py 40 records > $O/ncu_prof.log 2>&1; echo "ncu rc=$?" >> $O/ncu_prof.log
python scripts/ncu_summary.py $O/prof.ncu-rep $O/chunk40.json > $O/ncu_chunk40.json 2>&1
tail -4 $O/pytest_gpu.log $O/smoke.log $O/ncu_prof.log; cat $O/launch_summary.txt
for f in $O/bench*.log; do echo $f; grep "^{" $f | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln); print(d['value'], d['ms_per_step'], d.get('feasible_per_step'), d.get('kernel_ms_per_step'), d['roofline'].get('frac'), d.get('modes'), d.get('e2e'), d.get('cpu_baseline'), d.get('clocks'))
"; grep -i "error\|rc=" $f; done
