#!/bin/bash
# N-GPU pass: NCCL parity (tests/test_gpu_multi.py) + bench at N (cyclic, libme join) and at 1
O=gpurun_out/${OUT:-r2_multi}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 800 > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus $N --steps 5 --warmup 3 --no-cpu > $O/bench_n$N.log 2>&1; echo "rc=$?" >> $O/bench_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 \
  bench.py --gpus $N --steps 5 --warmup 3 --no-cpu --no-e2e --no-modes --partition even > $O/bench_n${N}_even.log 2>&1; echo "rc=$?" >> $O/bench_n${N}_even.log
tail -n 3 $O/pytest_multi.log
for f in $O/bench*.log; do echo $f; grep "^{" $f | python -c "
import json,sys
for ln in sys.stdin:
    d=json.loads(ln); print(round(d['value']/1e9,1), 'Gcfg/s', round(d['ms_per_step'],1), 'ms', d.get('feasible_per_step'), d['config']['parallelism'], {k: (round(v['value']/1e9,1), round(v['ms_per_step'],1)) for k,v in (d.get('modes') or {}).items()}, d.get('e2e'))
"; grep -i "error\|rc=" $f | tail -3; done
