#!/bin/bash
# k_tcp ring depth (ITLUMM_TCP_STAGES) x removal switches at cfg5 (dense): is the skeleton RTT-bound?
TAG=${1:-st}
mkdir -p gpurun_out
L=gpurun_out/tcpst_$TAG.log
for st in 2 3 4 5; do
  for d in 0 55 63 7; do
    echo "stages=$st dbg=$d" >> $L
    ITLUMM_TCP_STAGES=$st ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
done
