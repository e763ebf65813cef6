#!/bin/bash
# SS=2 default: full GPU parity suite, then removal attribution and a trace at cfg5 (dense).
TAG=${1:-ss2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 -k "not one_cta_streamed" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
L=gpurun_out/tcprm_$TAG.log
for d in 0 1 2 4 32 7 39 55; do
  echo "dbg=$d" >> $L
  ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
done
echo "ss=1 ref" >> $L
ITLUMM_TCP_SS=1 timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv >> $L
timeout 300 python tools/tcp_trace.py cfg5 tc_dense > gpurun_out/tcptrace_$TAG.log 2>&1
