#!/bin/bash
mkdir -p gpurun_out/r2q
for d in 0 512 1 513 64 2 514; do echo "dbg=$d" >> gpurun_out/r2q/kb.txt; ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc,tc_dense --only acc --iters 10 >> gpurun_out/r2q/kb.txt 2>&1; done
ITLUMM_TCP_DBG=512 timeout 300 python tools/tcp_trace.py cfg5 tc > gpurun_out/r2q/trace512.txt 2>&1
