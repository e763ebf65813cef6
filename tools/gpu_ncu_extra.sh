#!/bin/bash
# ncu --set full of the two other kernels of the benched steps: the row encoder at cfg5 and the
# resident-LUT k_tc at cfg2 split-packed (each after the same command ran clean without ncu).
O=gpurun_out/ncu_extra
mkdir -p $O
C1="python tools/kbench.py --workload cfg5 --algos tc_pipe --only encode --iters 2 --no-graph"
timeout 600 $C1 > $O/plain_enc.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_encode_rows -s 3 -c 1 -o $O/cfg5_encode $C1 > $O/ncu_enc.log 2>&1
echo rc=$? >> $O/ncu_enc.log
C2="python tools/kbench.py --workload cfg2 --algos tc_pipe --only acc --iters 2 --no-graph --packed"
timeout 600 $C2 > $O/plain_ktc.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 3 -c 1 -o $O/cfg2_packed_ktc $C2 > $O/ncu_ktc.log 2>&1
echo rc=$? >> $O/ncu_ktc.log
tail -n 2 $O/ncu_enc.log $O/ncu_ktc.log
