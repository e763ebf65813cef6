#!/bin/bash
# Three K-blocks per ring slot (ITLUMM_TCP_SS=3, needs the direct-codes layout): parity and timings.
TAG=${1:-ss3}
mkdir -p gpurun_out
ITLUMM_TCP_SS=3 ITLUMM_TCP_CDIRECT=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -k "streamed or benched or mlp or small or edge" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
L=gpurun_out/ss3_$TAG.log
for cfgx in "2 0" "2 1" "3 1"; do
  set -- $cfgx
  for w in cfg5 cfg3_c128 cfg3_c64; do
    echo "ss=$1 cdirect=$2 $w" >> $L
    ITLUMM_TCP_SS=$1 ITLUMM_TCP_CDIRECT=$2 timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc,fused --iters 20 >> $L 2>&1
  done
  ITLUMM_TCP_SS=$1 ITLUMM_TCP_CDIRECT=$2 ITLUMM_TCP_DBG=55 timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
done
ITLUMM_TCP_SS=3 ITLUMM_TCP_CDIRECT=1 timeout 300 python tools/clock_probe.py cfg5 acc >> $L 2>&1
