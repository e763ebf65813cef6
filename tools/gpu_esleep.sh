#!/bin/bash
# (ITLUMM_TCP_ESLEEP existed only for this probe; not in the tree)
# k_tcp: idle epilogue warps sleep (ITLUMM_TCP_ESLEEP ns per ring slot of the item) before polling the
# accumulator-full barrier, so that they are not woken by every barrier event of the SM.
O=gpurun_out/esleep
mkdir -p $O
L=$O/kbench.log
for rep in 1 2; do
for e in 0 100 200 300 400; do
  for w in cfg5 cfg3_c128; do
    echo "esleep=$e $w" >> $L
    ITLUMM_TCP_ESLEEP=$e timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
done
done
grep -v "^\s*$" $L | cut -c1-200 | paste - -
