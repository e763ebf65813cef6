#!/bin/bash
# Which agent bounds the k_tcp skeleton?  Producers (16384) or the LUT loader (32768) taken out of the ring.
TAG=${1:-who}
mkdir -p gpurun_out
L=gpurun_out/tcpwho_$TAG.log
for d in 55 16439 32823 16384 32772 0; do
  echo "dbg=$d" >> $L
  ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
done
