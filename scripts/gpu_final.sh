#!/bin/bash
# the measurement pass of a round: tests, smoke, ncu captures of one chunk per mode (copied into profiles/ on the
# box first, so the bench line's int_issue comes from this build), bench (driver settings), launch list
O=gpurun_out/${OUT:-r2_final}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi > $O/smi.txt 2>&1; (nproc; lscpu | head -20) > $O/host.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
ME_CHECKED=1 timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -k "not multi_gpu" > $O/pytest_gpu_checked.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_checked.log
for spec in "40 records" "240 records" "40 count" "40 index"; do
  set -- $spec; C=$1; M=$2
  python scripts/profile_chunk.py $C $M > $O/chunk${C}_$M.json 2>&1
  timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:rowcount_kernel|fused_kernel" -c 2 \
    -o $O/prof${C}_$M python scripts/profile_chunk.py $C $M > $O/ncu_prof${C}_$M.log 2>&1; echo "ncu rc=$?" >> $O/ncu_prof${C}_$M.log
  python scripts/ncu_summary.py $O/prof${C}_$M.ncu-rep $O/chunk${C}_$M.json > $O/ncu_chunk${C}_$M.json 2>&1
done
cp $O/ncu_chunk40_records.json $O/ncu_chunk40.json
mkdir -p profiles/r2_final && cp $O/ncu_chunk*.json profiles/r2_final/
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-modes --no-verify > $O/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $O/ncu_launch.log
python scripts/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
tail -n 3 $O/pytest_gpu.log $O/pytest_gpu_checked.log $O/smoke.log; cat $O/launch_summary.txt | head -8
grep "^{" $O/bench.log | head -c 3000; echo; grep "^{" $O/bench_ref.log | head -c 600
