#!/bin/bash
# K0 (row-count kernel) change: GPU tests (+ checked build), COUNT / RECORDS / INDEX bench, ncu of the count-only K0
O=gpurun_out/${OUT:-r2_k0}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 1400 ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -n 3 $O/pytest_gpu.log
if [ -n "$CHECKED" ]; then
  ME_CHECKED=1 timeout 1500 python -m pytest tests -m gpu -x -q --timeout 1400 -k "not multi_gpu" > $O/pytest_gpu_checked.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_checked.log
  tail -n 2 $O/pytest_gpu_checked.log
fi
OUT=${OUT:-r2_k0} MODES="count records index" VARIANTS="${VARIANTS:-ME_NONE=0}" bash scripts/gpu_ab_modes.sh
OUT=${OUT:-r2_k0}/prof PMODE=count bash scripts/gpu_prof_chunk.sh
