#!/bin/bash
# (the ITLUMM_TCP_FAST / ITLUMM_TCP_POLL switches exist only in commit b39554f; removed afterwards)
# k_tcp: who polls the barriers (ITLUMM_TCP_POLL bits: 1 producers, 2 epilogue, 4 MMA warp poll with
# lane 0 only) x producer loop (ITLUMM_TCP_FAST), accumulate only (kbench), one box.
O=gpurun_out/tcppoll
mkdir -p $O
L=$O/kbench.log
for f in 0 1; do
for p in 0 1 2 3 4 7; do
  for w in cfg5 cfg3_c128; do
    echo "fast=$f poll=$p $w" >> $L
    ITLUMM_TCP_FAST=$f ITLUMM_TCP_POLL=$p timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
done
done
grep -v "^\s*$" $L | cut -c1-200 | paste - - 
