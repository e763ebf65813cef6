#!/bin/bash
# k_tcp: codes straight from global memory (ITLUMM_TCP_CDIRECT, ring one slot deeper) x SS; parity.
TAG=${1:-cd}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -k "(streamed or cfg5 or cfg3 or mlp or edge or small) and not sel and not one_cta" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
L=gpurun_out/tcpcd_$TAG.log
for ss in 2 1; do
 for cd in 1 0; do
  for d in 0 55; do
    echo "ss=$ss cdirect=$cd dbg=$d" >> $L
    ITLUMM_TCP_SS=$ss ITLUMM_TCP_CDIRECT=$cd ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
 done
done
for w in cfg3_c128 cfg3_c64; do
 for cd in 1 0; do
  echo "cdirect=$cd $w" >> $L
  ITLUMM_TCP_CDIRECT=$cd timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc,fused --iters 20 >> $L 2>&1
 done
done
timeout 300 python tools/tcp_trace.py cfg5 tc_dense > gpurun_out/tcptrace_$TAG.log 2>&1
