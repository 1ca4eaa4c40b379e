#!/bin/bash
# the GPU tests against libme_checked.so (device-side bounds assertions: every
# table, scratch, shared-memory and output index the kernels compute; K3 finds
# exactly the survivors K0 counted).  compute-sanitizer is closed on the pool.
O=gpurun_out/${OUT:-r2_checked}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
ME_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -k "not multi_gpu" ${PYTEST_ARGS} > $O/pytest_checked.log 2>&1; echo "rc=$?" >> $O/pytest_checked.log
ME_CHECKED=1 timeout 600 python scripts/sanitize.py > $O/sanitize_checked.log 2>&1; echo "rc=$?" >> $O/sanitize_checked.log
ME_CHECKED=1 ME_MAX_ROWS=1 timeout 600 python scripts/sanitize.py > $O/sanitize_checked_rows1.log 2>&1; echo "rc=$?" >> $O/sanitize_checked_rows1.log
tail -n 3 $O/pytest_checked.log $O/sanitize_checked.log $O/sanitize_checked_rows1.log
