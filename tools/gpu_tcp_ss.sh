#!/bin/bash
# k_tcp: two K-blocks per ring slot (ITLUMM_TCP_SS=2) vs one; parity with SS=2, timings at cfg5/cfg3.
TAG=${1:-ss}
mkdir -p gpurun_out
L=gpurun_out/tcpss_$TAG.log
ITLUMM_TCP_SS=2 timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -x -k "(streamed or cfg5 or cfg3 or mlp) and not one_cta_streamed" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
for ss in 1 2; do
 for g in 0 1 2; do
  for d in 0 55; do
    echo "ss=$ss group=$g dbg=$d" >> $L
    ITLUMM_TCP_SS=$ss ITLUMM_TCP_GROUP=$g ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
 done
 for w in cfg3_c128 cfg3_c64; do
  echo "ss=$ss $w" >> $L
  ITLUMM_TCP_SS=$ss timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc,fused --iters 20 >> $L 2>&1
 done
done
ITLUMM_TCP_SS=2 timeout 300 python tools/tcp_trace.py cfg5 tc_dense > gpurun_out/tcptrace_$TAG.log 2>&1
