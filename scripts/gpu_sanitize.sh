#!/bin/bash
# compute-sanitizer over scripts/sanitize.py (every kernel path on small spaces)
O=gpurun_out/${OUT:-r2_sanitize}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  envs='"" ME_MAX_ROWS=1 ME_SERIAL=1'
  [ $tool = synccheck ] || [ $tool = initcheck ] && envs='""'
  for env in $(eval echo $envs); do
    tag=${tool}${env:+_$env}
    env $env timeout 1200 $CS --tool $tool --error-exitcode 9 python scripts/sanitize.py > $O/$tag.log 2>&1
    echo "$tag rc=$?" | tee -a $O/summary.txt
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE" $O/$tag.log | tail -3 >> $O/summary.txt
  done
done
cat $O/summary.txt
