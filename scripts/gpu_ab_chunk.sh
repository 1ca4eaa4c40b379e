#!/bin/bash
# bench A/B over the sweep call size and K3 stream alternation (records, N = 1)
O=gpurun_out/${OUT:-r2_abc}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for spec in ${SPECS:-"28 ME_NONE=0"}; do
  k=${spec%%:*}; v=${spec#*:}
  env $v timeout 600 python bench.py --chunk-log2 $k --steps 5 --warmup 3 --no-cpu --no-e2e --no-modes ${BARGS} > $O/bench_${k}_$v.log 2>&1
  echo "$k $v $(grep '^{' $O/bench_${k}_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,1), "Gcfg/s", round(d["ms_per_step"],1), "ms", {k: round(v,1) for k,v in d["kernel_ms_per_step"].items()})')"
done
