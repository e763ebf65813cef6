#!/bin/bash
mkdir -p gpurun_out/r2l
for d in 39 103 167 231 295 0 64 128 192 256; do echo "dbg=$d" >> gpurun_out/r2l/kbench.txt; ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc,tc_dense --only acc --iters 10 >> gpurun_out/r2l/kbench.txt 2>&1; done
