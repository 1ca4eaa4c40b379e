#!/bin/bash
# multi-GPU: GPU tests incl. the torchrun parity test, bench at N=1 and N=#GPUs
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -k "multi_gpu or next or stage" > gpurun_out/pytest_multi.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_multi.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/bench_n1.log 2>&1; echo "bench1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 3 --warmup 2 > gpurun_out/bench_n$NG.log 2>&1; echo "benchN rc=$?"
for f in gpurun_out/bench_n1.log gpurun_out/bench_n$NG.log; do python3 -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], '%.3e'%d['value'], '%.1f ms'%d['ms_per_step'], {k:round(v,1) for k,v in d['kernel_ms_per_step'].items()}, d.get('e2e',{}).get('value'), d.get('cpu_baseline',{}).get('value'))"; done
