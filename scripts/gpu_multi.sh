#!/bin/bash
# microbench + GPU tests (incl. multi-GPU) + bench at N=1 and N=#GPUs
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
./scripts/microbench > gpurun_out/microbench.json 2>&1 || (nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/microbench scripts/microbench.cu && ./scripts/microbench > gpurun_out/microbench.json 2>&1)
cat gpurun_out/microbench.json
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_n1.log 2>&1; echo "bench1 rc=$?"
tail -c 1500 gpurun_out/bench_n1.log
if [ "$NG" -ge 2 ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 3 --warmup 2 > gpurun_out/bench_n$NG.log 2>&1; echo "benchN rc=$?"
tail -c 1500 gpurun_out/bench_n$NG.log
fi
