#!/bin/bash
# K0: RECORDS / INDEX with the sorted-u lists in L1-cached global memory vs shared; ncu of the count-only K0 both ways
O=gpurun_out/${OUT:-r2_k0b}; mkdir -p $O
OUT=${OUT:-r2_k0b} MODES="records index" VARIANTS="ME_K0_SMEM=0 ME_K0_SMEM=1" bash scripts/gpu_ab_modes.sh
for v in 0 1; do
  ME_K0_SMEM=$v OUT=${OUT:-r2_k0b}/smem$v PMODE=count bash scripts/gpu_prof_chunk.sh
done
