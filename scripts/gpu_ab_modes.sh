#!/bin/bash
# A/B of launch knobs per output mode (bench.py, N = 1, 5 steps)
O=gpurun_out/${OUT:-r2_ab}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for mode in ${MODES:-index records}; do
  for v in ${VARIANTS:-ME_NONE=0}; do
    env $v timeout 600 python bench.py --mode $mode --steps 5 --warmup 3 --no-cpu --no-e2e --no-modes > $O/bench_${mode}_$v.log 2>&1
    echo "$mode $v $(grep '^{' $O/bench_${mode}_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,1), "Gcfg/s", round(d["ms_per_step"],1), "ms", {k: round(v,1) for k,v in d["kernel_ms_per_step"].items()})')"
  done
done
