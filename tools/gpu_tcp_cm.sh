#!/bin/bash
# Is the tcgen05.commit rate what bounds the k_tcp skeleton?  dbg 55 (skeleton) vs 55|8192 (plain arrivals).
TAG=${1:-cm}
mkdir -p gpurun_out
L=gpurun_out/tcpcm_$TAG.log
for ss in 2 1; do
  for d in 55 8247 2 8194; do
    echo "ss=$ss dbg=$d" >> $L
    ITLUMM_TCP_SS=$ss ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
done
