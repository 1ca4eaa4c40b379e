#!/bin/bash
# one ncu --set full capture of one C5 chunk (count + write kernels), after the
# same command ran clean without ncu
mkdir -p gpurun_out
python scripts/profile_chunk.py ${PCHUNK:-40} ${PMODE:-records} > gpurun_out/chunk40.json 2>&1 || { cat gpurun_out/chunk40.json; exit 1; }
cat gpurun_out/chunk40.json
timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:${PKERN:-count_kernel|write_kernel|stage_kernel|expand_kernel|row_kernel}" -c ${PCOUNT:-4} \
  -o gpurun_out/prof python scripts/profile_chunk.py ${PCHUNK:-40} ${PMODE:-records} > gpurun_out/ncu_prof.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_prof.log
