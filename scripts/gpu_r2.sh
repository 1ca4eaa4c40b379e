#!/bin/bash
# round-2 GPU pass: tests, smoke, bench of the row-count pipeline (pipe 3) vs the descriptor pipeline (pipe 2)
mkdir -p gpurun_out/r2
O=gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_p3.log 2>&1; echo "rc=$?" >> $O/bench_p3.log
ME_PIPE=2 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_p2.log 2>&1; echo "rc=$?" >> $O/bench_p2.log
for m in index count; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --mode $m > $O/bench_p3_$m.log 2>&1; echo "rc=$?" >> $O/bench_p3_$m.log; done
tail -5 $O/pytest_gpu.log $O/smoke.log
for f in $O/bench_*.log; do echo $f; python - "$f" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); print(d["value"], d["ms_per_step"], d.get("feasible_per_step"), d.get("kernel_ms_per_step"), d["roofline"].get("frac"))
    elif "rc=" in ln or "Error" in ln: print(ln.strip())
PY
done
