#!/bin/bash
# A/B of alternative builds (exp/libme_*.so) against the default build, per output mode (bench.py, N = 1, 5 steps)
O=gpurun_out/${OUT:-r2_ablibs}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
cp paper_2411_06465_b200/libme.so $O/libme.default
for l in default ${LIBS}; do
  if [ $l = default ]; then cp $O/libme.default paper_2411_06465_b200/libme.so; else cp exp/libme_$l.so paper_2411_06465_b200/libme.so; fi
  for mode in ${MODES:-records index}; do
    timeout 600 python bench.py --mode $mode --steps 5 --warmup 3 --no-cpu --no-e2e --no-modes --no-verify > $O/bench_${mode}_$l.log 2>&1
    echo "$l $mode $(grep '^{' $O/bench_${mode}_$l.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,1), "Gcfg/s", round(d["ms_per_step"],1), "ms", {k: round(v,1) for k,v in d["kernel_ms_per_step"].items()})')"
  done
done
cp $O/libme.default paper_2411_06465_b200/libme.so
