#!/bin/bash
# cfg2: is the k_tc tail (938 items on 148 SMs = 6.34 rounds) visible?  Accumulate at 60000 rows vs
# 56832 rows (888 items = 6 full rounds) vs 37888 (592 = 4 rounds); ncu of the packed encoder.
TAG=${1:-tail}
mkdir -p gpurun_out
L=gpurun_out/tail_$TAG.log
for n in 60000 56832 47360 37888; do
  timeout 300 python tools/kbench.py --workload cfg2 --packed --rows $n --algos tc_pipe --only encode,acc,fused --iters 50 >> $L 2>&1
done
CMD="python tools/kbench.py --workload cfg2 --packed --algos tc_pipe --only encode --iters 3 --no-graph"
timeout 300 $CMD > gpurun_out/tail_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:k_encode -s 4 -c 1 -o gpurun_out/enc_cfg2p $CMD > gpurun_out/tail_ncu.log 2>&1
echo rc=$? >> gpurun_out/tail_ncu.log
