O=gpurun_out/r2_final_launch; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-modes --no-verify > $O/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $O/ncu_launch.log
python scripts/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1; cat $O/launch_summary.txt
