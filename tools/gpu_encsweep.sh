#!/bin/bash
# Packed cfg2 encoder: stage size x bytes in flight (developer knobs), encode and full-call times.
TAG=${1:-es}
mkdir -p gpurun_out
L=gpurun_out/encsweep_$TAG.log
for kb in 8 16 24 48; do
  for inf in 50 100 150 200; do
    echo "stage_kb=$kb inflight_kb=$inf" >> $L
    ITLUMM_ENC_STAGE_KB=$kb ITLUMM_ENC_INFLIGHT_KB=$inf timeout 300 python tools/kbench.py --workload cfg2 --packed --algos tc_pipe --only encode,fused --iters 100 >> $L 2>&1
  done
done
