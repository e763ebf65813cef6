#!/bin/bash
# Wave quantisation of the resident-LUT k_tc at cfg2: 2 slices x ceil(N/128) tiles over 148 CTAs.
# N = 56832 is exactly 6 rounds, 60000 is 6.34 (runs 7), 66304 exactly 7.
O=gpurun_out/wave
mkdir -p $O
for n in 56832 60000 66304; do
  echo "rows=$n" >> $O/wave.log
  timeout 300 python tools/kbench.py --workload cfg2 --algos tc_pipe --only acc,fused --iters 50 --rows $n --packed >> $O/wave.log 2>&1
done
cat $O/wave.log | cut -c1-300
