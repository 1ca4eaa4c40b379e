#!/bin/bash
# count-only K0 variants: knobs on the default build, then alternative builds (exp/libme_*.so)
O=gpurun_out/${OUT:-r2_k0c}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
cp paper_2411_06465_b200/libme.so $O/libme.default
run() {  # name
  timeout 600 python bench.py --mode count --steps 5 --warmup 3 --no-cpu --no-e2e --no-modes > $O/bench_count_$1.log 2>&1
  echo "$1 $(grep '^{' $O/bench_count_$1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,1), "Gcfg/s", round(d["ms_per_step"],1), "ms", {k: round(v,1) for k,v in d["kernel_ms_per_step"].items()})')"
}
for v in ${VARIANTS:-ME_NONE=0}; do env $v bash -c "$(declare -f run); O=$O run $v"; done
for l in ${LIBS:-}; do cp exp/libme_$l.so paper_2411_06465_b200/libme.so; run $l; done
cp $O/libme.default paper_2411_06465_b200/libme.so
