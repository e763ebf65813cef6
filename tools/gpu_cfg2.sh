#!/bin/bash
TAG=${1:-c2}
mkdir -p gpurun_out
L=gpurun_out/cfg2_$TAG.log
timeout 300 python tools/kbench.py --workload cfg2 --packed --algos tc,tc_pipe,simt --only encode,acc,fused --iters 50 >> $L 2>&1
timeout 300 python tools/kbench.py --workload cfg2 --algos tc,tc_pipe --only encode,acc,fused --iters 50 >> $L 2>&1
ITLUMM_TC_NS_MAX=128 timeout 300 python tools/kbench.py --workload cfg2 --packed --algos tc,tc_pipe --only acc,fused --iters 50 >> $L 2>&1
