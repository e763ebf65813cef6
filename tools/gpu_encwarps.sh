#!/bin/bash
# Encoder consumer warps (ITLUMM_ENC_WARPS) x stage size on packed and row-major inputs.
TAG=${1:-ew}
mkdir -p gpurun_out
L=gpurun_out/encwarps_$TAG.log
for w in 8 12 16 24; do
  for kb in 24 48; do
    echo "warps=$w stage_kb=$kb" >> $L
    ITLUMM_ENC_WARPS=$w ITLUMM_ENC_STAGE_KB=$kb timeout 300 python tools/kbench.py --workload cfg2 --packed --algos tc_pipe --only encode,fused --iters 100 >> $L 2>&1
    ITLUMM_ENC_WARPS=$w ITLUMM_ENC_STAGE_KB=$kb timeout 300 python tools/kbench.py --workload cfg2 --algos tc_pipe --only encode,fused --iters 100 >> $L 2>&1
    ITLUMM_ENC_WARPS=$w ITLUMM_ENC_STAGE_KB=$kb timeout 300 python tools/kbench.py --workload cfg3_c128 --packed --algos tc_pipe --only encode,fused --iters 50 >> $L 2>&1
  done
done
for w in 8 16; do
  echo "warps=$w cfg5" >> $L
  ITLUMM_ENC_WARPS=$w timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe --only encode --iters 10 >> $L 2>&1
done
