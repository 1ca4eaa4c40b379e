#!/bin/bash
# K3 change: GPU parity (+ checked), RECORDS / INDEX bench, ncu of the sparse chunk 240
O=gpurun_out/${OUT:-r2_k3}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 1400 ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -n 2 $O/pytest_gpu.log
ME_CHECKED=1 timeout 1500 python -m pytest tests -m gpu -x -q --timeout 1400 -k "${PYTEST_K:-not multi_gpu}" > $O/pytest_gpu_checked.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_checked.log
tail -n 2 $O/pytest_gpu_checked.log
OUT=${OUT:-r2_k3} MODES="records index" VARIANTS="${VARIANTS:-ME_NONE=0}" bash scripts/gpu_ab_modes.sh
OUT=${OUT:-r2_k3}/prof PCHUNK=240 PMODE=records bash scripts/gpu_prof_chunk.sh
