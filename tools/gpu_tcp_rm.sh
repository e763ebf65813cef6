#!/bin/bash
# k_tcp removal attribution at cfg5 (dense and selector one-hot), developer switches ITLUMM_TCP_DBG.
TAG=${1:-rm}
mkdir -p gpurun_out
for m in dense sel; do
  for d in 0 1 2 4 32 7 39 55; do
    echo "mode=$m dbg=$d" >> gpurun_out/tcprm_$TAG.log
    ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_$m --only acc --iters 10 >> gpurun_out/tcprm_$TAG.log 2>&1
  done
done
timeout 300 python tools/tcp_trace.py cfg5 tc_dense > gpurun_out/tcptrace_$TAG.log 2>&1
