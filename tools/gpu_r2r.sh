#!/bin/bash
mkdir -p gpurun_out/r2r
CMD="python tools/kbench.py --workload cfg5 --algos tc --only acc --iters 2 --no-graph"
timeout 300 $CMD > gpurun_out/r2r/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcp -s 2 -c 1 -o gpurun_out/r2r/tcp_cfg5 $CMD > gpurun_out/r2r/ncu.log 2>&1
echo rc=$? >> gpurun_out/r2r/ncu.log
