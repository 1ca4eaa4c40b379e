#!/bin/bash
# ncu --set full of K0 + K3 on one C5 chunk (PCHUNK, default 40; PMODE records|index|full|count)
O=gpurun_out/${OUT:-r2_prof}; mkdir -p $O
C=${PCHUNK:-40}; M=${PMODE:-records}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python scripts/profile_chunk.py $C $M > $O/chunk$C.json 2>&1 || { cat $O/chunk$C.json; exit 1; }
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:rowcount_kernel|fused_kernel" -c 2 \
  -o $O/prof$C python scripts/profile_chunk.py $C $M > $O/ncu_prof$C.log 2>&1; echo "ncu rc=$?" >> $O/ncu_prof$C.log
python scripts/ncu_summary.py $O/prof$C.ncu-rep $O/chunk$C.json > $O/ncu_chunk$C.json 2>&1
cat $O/ncu_chunk$C.json | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d['kernels'].items(): print(k, {x: v[x] for x in ('duration_ms','dram_bytes_write','issue_frac','warps_active_pct','regs','top_stalls')})"
