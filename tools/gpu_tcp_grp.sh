#!/bin/bash
# k_tcp MMA-issue grouping (ITLUMM_TCP_GROUP) at cfg5 and cfg3 C=128: accumulate timings, skeleton, trace.
TAG=${1:-grp}
mkdir -p gpurun_out
L=gpurun_out/tcpgrp_$TAG.log
for g in 0 1 2 3 4; do
  for d in 0 55; do
    echo "group=$g dbg=$d" >> $L
    ITLUMM_TCP_GROUP=$g ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense,tc_pipe_sel --only acc --iters 10 >> $L 2>&1
  done
done
for g in 0 2 4; do
  echo "group=$g cfg3_c128" >> $L
  ITLUMM_TCP_GROUP=$g timeout 300 python tools/kbench.py --workload cfg3_c128 --algos tc_pipe_dense --only acc,fused --iters 20 >> $L 2>&1
done
ITLUMM_TCP_GROUP=2 timeout 300 python tools/tcp_trace.py cfg5 tc_dense > gpurun_out/tcptrace_$TAG.log 2>&1
