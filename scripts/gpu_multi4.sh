#!/bin/bash
# all GPU tests (incl. the torchrun multi-GPU parity), bench at N = 2 and N = #GPUs
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1500 > gpurun_out/pytest_multi.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_multi.log
for n in 2 $NG; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_n$n.log 2>&1; echo "bench$n rc=$?"
python3 -c "
import json,sys; d=json.loads(open('gpurun_out/bench_n$n.log').read().strip().splitlines()[-1]); print('N=$n', d['n_gpus'], '%.3e'%d['value'], '%.1f ms'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()}, d.get('e2e',{}).get('value'))"
done
