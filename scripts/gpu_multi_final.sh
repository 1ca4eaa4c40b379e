#!/bin/bash
# N-GPU pass at HEAD: the whole GPU suite (NCCL parity at N ranks included) + bench at N (cyclic, libme join) and even
O=gpurun_out/${OUT:-r2_multi_final}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 1400 > $O/pytest_gpu_n$N.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_n$N.log
OUT=${OUT:-r2_multi_final} bash scripts/gpu_multi_r2.sh
tail -n 3 $O/pytest_gpu_n$N.log
