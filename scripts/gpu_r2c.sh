#!/bin/bash
# quick iteration: GPU tests + bench (records, serial comparison)
O=gpurun_out/${OUT:-r2c}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS} > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
for v in ${VARIANTS}; do env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-modes > $O/bench_$v.log 2>&1; echo "rc=$?" >> $O/bench_$v.log; done
tail -n 4 $O/pytest_gpu.log
for f in $O/bench*.log; do echo $f; grep "^{" $f | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln); print(round(d['value']/1e9,1), 'Gcfg/s', round(d['ms_per_step'],1), 'ms', d.get('feasible_per_step'), {k: round(v,1) for k,v in d.get('kernel_ms_per_step').items()}, round(d['roofline'].get('frac') or 0,3), {k: (round(v['value']/1e9,1), round(v['ms_per_step'],1)) for k,v in (d.get('modes') or {}).items()})
"; grep -i "error\|rc=" $f | tail -3; done
