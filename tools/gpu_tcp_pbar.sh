#!/bin/bash
# k_tcp: combined producer arrivals (ITLUMM_TCP_PBAR) x MMA grouping at cfg5 and cfg3 C=128; parity with PBAR=1.
TAG=${1:-pbar}
mkdir -p gpurun_out
L=gpurun_out/tcppbar_$TAG.log
ITLUMM_TCP_PBAR=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -x -k "streamed or cfg5 or cfg3" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
for pb in 0 1; do
 for g in 0 2; do
  for d in 0 55; do
    echo "pbar=$pb group=$g dbg=$d" >> $L
    ITLUMM_TCP_PBAR=$pb ITLUMM_TCP_GROUP=$g ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
 done
done
for pb in 0 1; do
  echo "pbar=$pb cfg3_c128" >> $L
  ITLUMM_TCP_PBAR=$pb timeout 300 python tools/kbench.py --workload cfg3_c128 --algos tc_pipe_dense --only acc,fused --iters 20 >> $L 2>&1
done
ITLUMM_TCP_PBAR=1 timeout 300 python tools/tcp_trace.py cfg5 tc_dense > gpurun_out/tcptrace_$TAG.log 2>&1
