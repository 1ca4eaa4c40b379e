#!/bin/bash
# N>1 bench: cyclic vs even partition of C5 (kernel-only legs)
mkdir -p gpurun_out
N=${1:-2}
for P in cyclic even cyclic; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu --partition $P > gpurun_out/part_${N}_$P.log 2>&1
  echo "$P rc=$?"; tail -1 gpurun_out/part_${N}_$P.log | cut -c1-400
done
