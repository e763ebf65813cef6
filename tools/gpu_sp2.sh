#!/bin/bash
# 2:4-sparse one-hot with two K-blocks per ring slot: parity, burst and sustained timings vs dense.
TAG=${1:-sp2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -k "sp24 or one_cta or benched" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
L=gpurun_out/sp2_$TAG.log
for w in cfg5 cfg3_c128 cfg3_c64; do
  timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense,tc_pipe_sp24 --only acc,fused --iters 20 >> $L 2>&1
done
