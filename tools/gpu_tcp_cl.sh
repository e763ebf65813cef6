#!/bin/bash
# k_tcp: codes loader warp (ITLUMM_TCP_CLOAD) x SS at cfg5/cfg3; streamed parity with the defaults.
TAG=${1:-cl}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -k "(streamed or cfg5 or cfg3 or mlp) and not sel and not one_cta" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
L=gpurun_out/tcpcl_$TAG.log
for ss in 2 1; do
 for cl in 1 0; do
  for d in 0 55; do
    echo "ss=$ss cload=$cl dbg=$d" >> $L
    ITLUMM_TCP_SS=$ss ITLUMM_TCP_CLOAD=$cl ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
 done
done
for w in cfg3_c128 cfg3_c64; do
 for cl in 1 0; do
  echo "cload=$cl $w" >> $L
  ITLUMM_TCP_CLOAD=$cl timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc,fused --iters 20 >> $L 2>&1
 done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv >> $L
