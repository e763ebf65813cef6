#!/bin/bash
mkdir -p gpurun_out/r2d
for w in cfg5 cfg3_c128; do timeout 300 python tools/kbench.py --workload $w --algos tc,tc_dense --only acc --iters 20 >> gpurun_out/r2d/kbench.jsonl 2>> gpurun_out/r2d/kbench.err; done
CMD="python tools/kbench.py --workload cfg3_c128 --algos tc --only acc --iters 2 --no-graph"
timeout 300 $CMD > gpurun_out/r2d/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcp -s 2 -c 1 -o gpurun_out/r2d/tcp_c128 $CMD > gpurun_out/r2d/ncu.log 2>&1
echo rc=$? >> gpurun_out/r2d/ncu.log
